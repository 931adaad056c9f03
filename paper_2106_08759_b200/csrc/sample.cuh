// sample.cuh -- seeded sampling of Small g and Short f, and the small-factor invertibility test.
//
// KeyGen step 1 / step 3 and Algorithm 1 lines 4-6: "g <-$ R/3",
// "if not isInvertible(g): continue", "f <-$ Short".  The paper does not fix the sampler; the
// conventions are DESIGN.md C2 (stream), C3 (Small), C4 (Short by sorting p tagged uint32 draws).
// isInvertible is split: factors of degree <= 64 are tested here with residue
// tables (g mod f_i = sum_j g_j * (x^j mod f_i)); every larger factor is covered exactly by the
// product-tree root test (divstep.cuh) plus the per-key repair path.
#pragma once
#include "common.cuh"

namespace sntrup {

// ---------------------------------------------------------------------------------------------
// Warp-wide bitonic sort of 32*E uint32 keys held in registers, blocked layout: lane l holds
// global elements l*E .. l*E+E-1 in v[0..E-1].  Ascending.  A fixed network (constant time).
// Variant with every comparator ascending: each merge stage starts with the "mirror" step
// (i <-> i ^ (k-1)) followed by half-cleaners (i <-> i ^ j), so no direction selects are needed.
// Comparators on the low log2(E) index bits are in-register (min + max).  For E >= 32 the merge
// stages with k >= 4E transpose the warp's keys through shared memory into the striped layout
// (lane L holds elements r*32 + L in v[r]), where every index bit >= 5 is a register bit: the
// mirror is one SHFL per key and the half-cleaners with j >= 32 are in-register; the transpose
// back then leaves j < 32 in registers again.  (The blocked-only network spends a SHFL and a
// per-lane min/max select per key on each of its 15 cross-lane stages at E = 32.)
// Shared memory: 4 warps per block (all callers launch 128 threads).
// ---------------------------------------------------------------------------------------------
// Padded shared-memory index for the blocked <-> striped transposes: rows of 32 keys padded to
// 36 words (16-byte aligned blocked accesses, conflict-free striped accesses).
__device__ __forceinline__ int sort_pad(int i) { return i + 4 * (i >> 5); }

// One merge stage (k = 2^LS) of warp_bitonic_sort, as a template so that every index is a
// compile-time constant without relying on the unroller (E = 64 otherwise lands v in local memory).
// NR: keys at positions >= NR are pads (0xFFFFFFFF, above every real key); since every comparator
// puts the minimum at the lower position, pads never move and a comparator whose upper position
// is a pad is a no-op -- in the striped layout, registers r >= RP hold only pads and such
// comparators (and their transposes) are skipped at compile time.
template <int E, int LS, int NR>
__device__ __forceinline__ void bitonic_merge_stage(uint32_t (&v)[E], int lane, uint32_t *buf) {
    constexpr int k = 1 << LS;
    constexpr int RP = (NR + 31) / 32;                    // striped registers holding a real key
    constexpr bool TRANSPOSE = E >= 32;
    constexpr bool STRIPED = TRANSPOSE && k >= 4 * E;
    constexpr int JTOP = STRIPED ? 16 : k >> 2;           // first half-cleaner in blocked layout
    if constexpr (k <= E) {
        // mirror step, in-register
#pragma unroll
        for (int e = 0; e < E; e++) {
            const int ex = e ^ (k - 1);
            if ((e & (k >> 1)) == 0) {
                const uint32_t a = v[e], b = v[ex];
                v[e] = min(a, b);
                v[ex] = max(a, b);
            }
        }
    } else if constexpr (!STRIPED) {
        // mirror step across lanes (blocked): partner lane = lane ^ lm, element E-1-e
        constexpr int lm = k / E - 1;
        const bool lower = (lane & ((k / E) >> 1)) == 0;
        uint32_t o[E];
#pragma unroll
        for (int e = 0; e < E; e++) o[e] = __shfl_xor_sync(FULL, v[E - 1 - e], lm);
#pragma unroll
        for (int e = 0; e < E; e++) v[e] = lower ? min(v[e], o[e]) : max(v[e], o[e]);
    } else {
        // to striped: lane L holds elements 32 r + L in v[r]
        __syncwarp();
#pragma unroll
        for (int e = 0; e < E; e += 4)
            *reinterpret_cast<uint4 *>(&buf[sort_pad(lane * E + e)]) = make_uint4(v[e], v[e + 1], v[e + 2], v[e + 3]);
        __syncwarp();
#pragma unroll
        for (int r = 0; r < E; r++) v[r] = r < RP ? buf[sort_pad(32 * r + lane)] : 0xFFFFFFFFu;
        // mirror: partner lane ^ 31, register r ^ rm; lower half (r & rh) == 0
        constexpr int rm = (k - 1) >> 5, rh = k >> 6;
#pragma unroll
        for (int r = 0; r < E; r++) {
            if ((r & rh) == 0 && (r ^ rm) < RP) {
                const uint32_t a = __shfl_xor_sync(FULL, v[r ^ rm], 31);
                const uint32_t b = __shfl_xor_sync(FULL, v[r], 31);
                v[r] = min(v[r], a);
                v[r ^ rm] = max(v[r ^ rm], b);
            }
        }
        // half-cleaners j = k/4 .. 32: register bit j/32
#pragma unroll
        for (int jr = k >> 7; jr >= 1; jr >>= 1) {
#pragma unroll
            for (int r = 0; r < E; r++) {
                if ((r & jr) == 0 && (r | jr) < RP) {
                    const uint32_t a = v[r], b = v[r | jr];
                    v[r] = min(a, b);
                    v[r | jr] = max(a, b);
                }
            }
        }
        // back to blocked
        __syncwarp();
#pragma unroll
        for (int r = 0; r < RP && r < E; r++) buf[sort_pad(32 * r + lane)] = v[r];   // pads stay in buf
        __syncwarp();
#pragma unroll
        for (int e = 0; e < E; e += 4) {
            const uint4 q = *reinterpret_cast<const uint4 *>(&buf[sort_pad(lane * E + e)]);
            v[e] = q.x; v[e + 1] = q.y; v[e + 2] = q.z; v[e + 3] = q.w;
        }
    }
    // half-cleaners j = JTOP .. 1 (blocked layout)
#pragma unroll
    for (int j = JTOP; j >= 1; j >>= 1) {
        if (j >= E) {
            const int lm = j / E;
            const bool lower = (lane & lm) == 0;
#pragma unroll
            for (int e = 0; e < E; e++) {
                const uint32_t o = __shfl_xor_sync(FULL, v[e], lm);
                v[e] = lower ? min(v[e], o) : max(v[e], o);
            }
        } else {
#pragma unroll
            for (int e = 0; e < E; e++) {
                if ((e & j) == 0) {
                    const uint32_t a = v[e], b = v[e | j];
                    v[e] = min(a, b);
                    v[e | j] = max(a, b);
                }
            }
        }
    }
}

template <int E, int NR = 32 * E>
__device__ __forceinline__ void warp_bitonic_sort(uint32_t (&v)[E], int lane) {
    constexpr int N = 32 * E;
    constexpr int LE = E == 8 ? 3 : E == 16 ? 4 : E == 32 ? 5 : E == 64 ? 6 : -1;
    constexpr int LOGN = LE + 5;
    static_assert(LE > 0, "E must be 8, 16, 32 or 64");
    __shared__ __align__(16) uint32_t tb[4][E >= 32 ? N + N / 8 : 4];
    uint32_t *buf = tb[(threadIdx.x >> 5) & 3];
    bitonic_merge_stage<E, 1, NR>(v, lane, buf);
    bitonic_merge_stage<E, 2, NR>(v, lane, buf);
    bitonic_merge_stage<E, 3, NR>(v, lane, buf);
    bitonic_merge_stage<E, 4, NR>(v, lane, buf);
    bitonic_merge_stage<E, 5, NR>(v, lane, buf);
    bitonic_merge_stage<E, 6, NR>(v, lane, buf);
    bitonic_merge_stage<E, 7, NR>(v, lane, buf);
    bitonic_merge_stage<E, 8, NR>(v, lane, buf);
    if constexpr (LOGN >= 9) bitonic_merge_stage<E, 9, NR>(v, lane, buf);
    if constexpr (LOGN >= 10) bitonic_merge_stage<E, 10, NR>(v, lane, buf);
    if constexpr (LOGN >= 11) bitonic_merge_stage<E, 11, NR>(v, lane, buf);
}

// C4: Short f for key root K (domain d = 0).  Writes the int8 row f[0..P16).
template <class PS>
__device__ __forceinline__ void sample_short_warp(uint64_t K, int8_t *frow, int lane, uint64_t domain = 0) {
    constexpr int E = PS::NSORT / 32;
    const uint64_t D = sm_at(K, domain);
    uint32_t v[E];
#pragma unroll
    for (int t = 0; t < E / 2; t++) {
        const int i = lane * E + 2 * t;                     // words u_i (low half), u_{i+1} (high)
        const uint64_t z = sm_at(D, (uint64_t)(i / 2));
        const uint32_t lo = (uint32_t)z, hi = (uint32_t)(z >> 32);
        v[2 * t] = i < PS::P ? (i < PS::W ? (lo & 0xFFFFFFFEu) : ((lo & 0xFFFFFFFCu) | 1u))
                             : 0xFFFFFFFFu;
        v[2 * t + 1] = i + 1 < PS::P ? (i + 1 < PS::W ? (hi & 0xFFFFFFFEu)
                                                      : ((hi & 0xFFFFFFFCu) | 1u))
                                     : 0xFFFFFFFFu;
    }
    warp_bitonic_sort<E, PS::P>(v, lane);
    // f_i = (L_(i) & 3) - 1 for i < P, 0 in the pad; pack 4 per word, 16-byte stores.
#pragma unroll
    for (int w4 = 0; w4 < E / 16; w4++) {
        const int base = lane * E + 16 * w4;
        if (base >= PS::P16) break;
        uint32_t wd[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
            uint32_t word = 0;
#pragma unroll
            for (int b = 0; b < 4; b++) {
                const int e = 16 * w4 + 4 * q + b;
                const int i = lane * E + e;
                word |= (i < PS::P ? (v[e] & 3u) : 1u) << (8 * b);   // f + 1 in {0,1,2}
            }
            // byte-wise (f + 1) - 1 without borrows: bytes are < 0x80.
            wd[q] = ((word | 0x80808080u) - 0x01010101u) ^ 0x80808080u;
        }
        *reinterpret_cast<uint4 *>(frow + base) = make_uint4(wd[0], wd[1], wd[2], wd[3]);
    }
}

// C3: Small g, attempt a (domain 1 + a) for block b (coefficients 32b .. 32b+31): bitsliced
// planes (pl, mi).  Coefficients >= P are 0.
template <class PS>
__device__ __forceinline__ void small_block(uint64_t D, int b, uint32_t &pl, uint32_t &mi) {
    pl = 0;
    mi = 0;
#pragma unroll 4
    for (int t = 0; t < 16; t++) {
        const int i = 32 * b + 2 * t;
        if (i >= PS::P) break;
        const uint64_t z = sm_at(D, (uint64_t)(i / 2));
        const uint32_t u0 = (uint32_t)z & 0x3FFFFFFFu, u1 = (uint32_t)(z >> 32) & 0x3FFFFFFFu;
        // c = (3 u) >> 30 in {0,1,2} -> g = c - 1 (3 u < 2^32): plus iff bit 31 is set, minus iff
        // c - 1 is negative.
        const uint32_t t0 = 3u * u0, t1 = 3u * u1;
        pl |= (t0 >> 31) << (2 * t);
        mi |= (((t0 >> 30) - 1u) >> 31) << (2 * t);
        if (i + 1 < PS::P) {
            pl |= (t1 >> 31) << (2 * t + 1);
            mi |= (((t1 >> 30) - 1u) >> 31) << (2 * t + 1);
        }
    }
}

// Write bitsliced block b to an int8 row (32 bytes; bytes beyond P16 are not written).
template <class PS>
__device__ __forceinline__ void store_block_int8(int8_t *row, int b, uint32_t pl, uint32_t mi) {
#pragma unroll
    for (int h = 0; h < 2; h++) {
        const int base = 32 * b + 16 * h;
        if (base >= PS::P16) break;
        uint32_t wd[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
            // SWAR: spread 4 plane bits to the 4 bytes (copies at shifts 0, 7, 14, 21 are disjoint),
            // then byte = +1 (pl) or 0xFF (mi); the planes are disjoint so no byte sees both.
            const int sh = 16 * h + 4 * q;
            const uint32_t P = (((pl >> sh) & 15u) * 0x00204081u) & 0x01010101u;
            const uint32_t M = (((mi >> sh) & 15u) * 0x00204081u) & 0x01010101u;
            wd[q] = P | (M * 0xFFu);
        }
        *reinterpret_cast<uint4 *>(row + base) = make_uint4(wd[0], wd[1], wd[2], wd[3]);
    }
}

// Load block b of an int8 row into bitsliced planes (coefficients >= P ignored).
template <class PS>
__device__ __forceinline__ void load_block_int8(const int8_t *row, int b, uint32_t &pl, uint32_t &mi) {
    pl = 0;
    mi = 0;
#pragma unroll
    for (int h = 0; h < 2; h++) {
        const int base = 32 * b + 16 * h;
        if (base >= PS::P16) break;
        const uint4 q4 = *reinterpret_cast<const uint4 *>(row + base);
        const uint32_t wd[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
        for (int q = 0; q < 4; q++)
#pragma unroll
            for (int c = 0; c < 4; c++) {
                const int bit = 16 * h + 4 * q + c;
                const int idx = base + 4 * q + c;
                const int val = (int)(int8_t)((wd[q] >> (8 * c)) & 0xffu);
                if (idx < PS::P) {
                    pl |= (uint32_t)(val == 1) << bit;
                    mi |= (uint32_t)(val == -1) << bit;
                }
            }
    }
}

// Small-factor residue test (warp).  T: [P][WT] uint2 rows (x^j mod f_i concatenated over the
// small factors, bitsliced); masks: [nf][WT] words selecting each factor's trits.  Blocks are
// distributed over lanes (block b on lane b % 32).  Returns true iff no small factor divides g.
// Constant time in g (reading Z19: only the attempt count may vary): every coefficient
// j < p adds T[j] selected by masks (+T[j] for g_j = 1, -T[j] for g_j = -1, 0 otherwise) -- the
// trip counts and every load address depend only on p, never on g.
template <class PS, int NBL>
__device__ __forceinline__ bool small_factor_check(const uint32_t (&pl)[NBL], const uint32_t (&mi)[NBL],
                                                   const uint2 *__restrict__ T,
                                                   const uint32_t *__restrict__ masks, int nf,
                                                   int lane) {
    constexpr int WT = PS::WT;
    uint32_t ap[WT], am[WT];
#pragma unroll
    for (int w = 0; w < WT; w++) { ap[w] = 0; am[w] = 0; }
    // lane L takes coefficients j = 32 c + L of every block c: the warp's T loads are coalesced
    // (consecutive rows), and block c's two planes are broadcast from its lane by two shuffles
#pragma unroll
    for (int c = 0; c < PS::NB32; c++) {
        const uint32_t bp = __shfl_sync(FULL, pl[c >> 5], c & 31);
        const uint32_t bm = __shfl_sync(FULL, mi[c >> 5], c & 31);
        const int j = 32 * c + lane;
        if (j < PS::P) {                                     // public: depends on p and the lane
            const uint32_t mp = 0u - ((bp >> lane) & 1u), mm = 0u - ((bm >> lane) & 1u);
#pragma unroll
            for (int w = 0; w < WT; w++) {
                const uint2 t = __ldg(&T[(size_t)j * WT + w]);
                // g_j T[j]: T[j] if g_j = 1, its negation (planes swapped) if g_j = -1, else 0
                gf3_add(ap[w], am[w], (t.x & mp) | (t.y & mm), (t.y & mp) | (t.x & mm));
            }
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
#pragma unroll
        for (int w = 0; w < WT; w++) {
            const uint32_t op = __shfl_xor_sync(FULL, ap[w], off);
            const uint32_t om = __shfl_xor_sync(FULL, am[w], off);
            gf3_add(ap[w], am[w], op, om);
        }
    // every factor's verdict computed (no early exit), combined without branches
    uint32_t all_ok = 1u;
    for (int f = 0; f < nf; f++) {
        uint32_t nz = 0;
#pragma unroll
        for (int w = 0; w < WT; w++) nz |= (ap[w] | am[w]) & masks[f * WT + w];
        all_ok &= (uint32_t)(nz != 0);
    }
    return all_ok != 0;
}

// ---------------------------------------------------------------------------------------------
// Sampling kernel: one warp per key.  f from domain 0; g from domains 1, 2, ... until the
// small-factor test passes (or the first draw when the test is disabled).
// ---------------------------------------------------------------------------------------------
struct SampleArgs {
    uint64_t seed, first, n;
    int8_t *G, *F;          // rows of P16 bytes
    uint8_t *attempts;
    const uint2 *T;
    const uint32_t *masks;
    int nf;
    int small_check;
    int *err;               // set if the retry bound is hit
};

template <class PS>
__global__ void __launch_bounds__(128) sample_kernel(SampleArgs a) {
    const int lane = threadIdx.x & 31;
    const uint64_t key_local = (uint64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    if (key_local >= a.n) return;
    const uint64_t K = sm_at(a.seed, a.first + key_local);
    sample_short_warp<PS>(K, a.F + key_local * PS::P16, lane);

    constexpr int NBL = (PS::NB32 + 31) / 32;
    uint32_t pl[NBL], mi[NBL];
    int attempt = 0;
    for (;;) {
        const uint64_t D = sm_at(K, 1 + (uint64_t)attempt);
#pragma unroll
        for (int s = 0; s < NBL; s++) {
            const int b = lane + 32 * s;
            if (b < PS::NB32) small_block<PS>(D, b, pl[s], mi[s]);
            else { pl[s] = 0; mi[s] = 0; }
        }
        if (!a.small_check) break;
        if (small_factor_check<PS, NBL>(pl, mi, a.T, a.masks, a.nf, lane)) break;
        if (++attempt >= 255) { if (lane == 0) atomicExch(a.err, 1); break; }
    }
    int8_t *grow = a.G + key_local * PS::P16;
#pragma unroll
    for (int s = 0; s < NBL; s++) {
        const int b = lane + 32 * s;
        if (32 * b < PS::P16) store_block_int8<PS>(grow, b, pl[s], mi[s]);
    }
    if (lane == 0 && a.attempts) a.attempts[key_local] = (uint8_t)(attempt + 1);
}

// Short elements of an arbitrary stream domain (C2: domain 0 = f; domains >= 2^32 reserved for
// encapsulation draws), one warp per global key index.
template <class PS>
__global__ void __launch_bounds__(128) short_kernel(uint64_t seed, uint64_t first, uint64_t n,
                                                    uint64_t domain, int8_t *out) {
    const int lane = threadIdx.x & 31;
    const uint64_t row = (uint64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    if (row >= n) return;
    sample_short_warp<PS>(sm_at(seed, first + row), out + row * PS::P16, lane, domain);
}

// SURVEY.md 8(c) C12 (BASELINE configs[2] inputs): uniform R/q element from stream domain
// `domain` of key root SM(seed, first + row): a_j = floor(u_j q / 2^32) - (q-1)/2, int16 rows of
// P8 (pad 0).  One thread per output word pair: thread t of the row computes SM(D, t) and writes
// coefficients 2t, 2t+1 (low word first, C2).
template <class PS>
__global__ void __launch_bounds__(128) uniform_rq_kernel(uint64_t seed, uint64_t first, uint64_t n,
                                                         uint64_t domain, int16_t *out) {
    constexpr int PAIRS = PS::P8 / 2;
    const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t row = gid / PAIRS;
    const int t = (int)(gid - row * PAIRS);
    if (row >= n) return;
    const uint64_t D = sm_at(sm_at(seed, first + row), domain);
    const uint64_t z = sm_at(D, (uint64_t)t);
    const uint32_t u0 = (uint32_t)z, u1 = (uint32_t)(z >> 32);
    const int a0 = 2 * t < PS::P ? (int)(((uint64_t)u0 * PS::Q) >> 32) - PS::QH : 0;
    const int a1 = 2 * t + 1 < PS::P ? (int)(((uint64_t)u1 * PS::Q) >> 32) - PS::QH : 0;
    reinterpret_cast<uint32_t *>(out + row * PS::P8)[t] = (uint32_t)(uint16_t)a0 | ((uint32_t)(uint16_t)a1 << 16);
}

// ok[row] = (number of nonzero coefficients of row == W) (decapsulation's weight check)
template <class PS>
__global__ void __launch_bounds__(128) weight_check_kernel(const int8_t *r, uint64_t n, uint8_t *ok) {
    const int lane = threadIdx.x & 31;
    const uint64_t row = (uint64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    if (row >= n) return;
    const uint4 *rr = reinterpret_cast<const uint4 *>(r + row * PS::P16);
    int cnt = 0;
    for (int c = lane; c < PS::P16 / 16; c += 32) {
        const uint4 q = rr[c];
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int i = 0; i < 4; i++) cnt += __popc(w[i] & 0x01010101u);   // nonzero trit <=> odd byte
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) cnt += __shfl_xor_sync(FULL, cnt, off);
    if (lane == 0) ok[row] = cnt == PS::W ? 1 : 0;
}

}  // namespace sntrup
