// tc4mul.cuh -- FP4 variant of the tensor-core ring product: tcgen05.mma kind::mxf4
// (block32 scale factors, all 2^0), for products with a small operand.
//
// Every operand digit is an integer in [-4, 4], exactly representable in e2m1
// ({0, 0.5, 1, 1.5, 2, 3, 4, 6}): small operands (R/3 elements, g, 3f in {-3, 0, 3}) are one
// digit; an R/q element is written in balanced base 9 (LB digits: 9^4 = 6561 covers q <= 6561,
// 5 digits above).  The A operand (the small one, Hankel) packs 64 K-elements into each 32-byte
// row slice, so every MMA reads half the A bytes of the int8 path per unit of K -- the
// shared-memory operand fetch that bounds tcmul.cuh.  Accumulation is fp32
// in TMEM: every sum is an integer of magnitude < 2^24 (|digit products| <= 16, K <= 1408),
// hence exact.  Same Hankel construction as tcmul.cuh at nibble granularity: window row rho =
// nibbles [rho, rho+32) of hA, SBO = 128 B (8 rows), LBO = 512 B (32 rows = one 32-element chunk).
#pragma once
#include "tcmul.cuh"

namespace sntrup {

__host__ __device__ constexpr int digits9(int q) {       // balanced base-9 digits covering |v| <= (q-1)/2
    int n = 1, cover = 4;
    while (cover < (q - 1) / 2) { cover = 9 * cover + 4; n++; }
    return n;
}

// e2m1 code of an integer in [-4, 4] or +-6
__device__ __forceinline__ uint32_t e2m1_code(int d) {
    const int a = d < 0 ? -d : d;
    return ((0x7065420u >> (4 * a)) & 0xFu) | (d < 0 ? 8u : 0u);   // |d| in {0..4, 6}
}

// SWAR e2m1 packing of 8 int8 coefficients in {-s, 0, s}, s in {1, 3} (bytes of w0 = coefficients
// 0..3, w1 = 4..7) into one word, nibble i = coefficient i.  Nonzero <=> byte bit 0 (1, 3, 0xff,
// 0xfd all odd); sign = byte bit 7; e2m1 magnitude code 2 (1.0) or 5 (3.0), sign bit 8.
__device__ __forceinline__ uint32_t e2m1_pack8_int8(uint32_t w0, uint32_t w1, int scale) {
    auto nib = [scale](uint32_t w) {
        const uint32_t m = w & 0x01010101u, s = (w >> 7) & 0x01010101u;
        const uint32_t mag = scale == 1 ? (m << 1) : ((m << 2) | m);
        uint32_t x = mag | (s << 3);                  // one nibble value per byte
        x = (x | (x >> 4)) & 0x00FF00FFu;
        return (x | (x >> 8)) & 0x0000FFFFu;
    };
    return nib(w0) | (nib(w1) << 16);
}

// e2m1 codes of x_i + y_i for nibble-packed x, y with values in {-s, 0, s} (s = 1: code 2;
// s = 3: code 5): sums in {0, +-s, +-2s}, 2s = 2.0 (code 4) or 6.0 (code 7).  Bitwise on the
// nonzero / sign bits of each nibble.
__device__ __forceinline__ uint32_t e2m1_pair_sum(uint32_t x, uint32_t y, int scale) {
    constexpr uint32_t M1 = 0x11111111u;
    const uint32_t nx = (scale == 1 ? x >> 1 : x) & M1, ny = (scale == 1 ? y >> 1 : y) & M1;
    const uint32_t sx = (x >> 3) & M1, sy = (y >> 3) & M1;
    const uint32_t same = nx & ny & ~(sx ^ sy), one = nx ^ ny;
    const uint32_t sg = ((nx & sx) | (ny & sy)) & (same | one);
    return same * (scale == 1 ? 4u : 7u) + one * (scale == 1 ? 2u : 5u) + (sg << 3);
}

// nibble order reversal of a word (nibble i -> nibble 7 - i)
__device__ __forceinline__ uint32_t nibble_reverse(uint32_t x) {
    const uint32_t y = __byte_perm(x, 0, 0x0123);
    return ((y >> 4) & 0x0F0F0F0Fu) | ((y << 4) & 0xF0F0F0F0u);
}

// TA > 0: the first NTA K steps of the Hankel A operand live in TMEM ([a-tmem] MMA form) instead
// of shared memory, within a TA-column allocation: every thread writes its own window row (TMEM
// lane r = output residue r) from registers with tcgen05.st, so those MMAs read only B from shared
// memory (scripts/probe/tmem_a_probe.cu: exact; 12.5 vs 39 cycles per M128 N16 K64 MMA per SM at 4
// CTAs).  The remaining K steps read shared-memory windows as before.
template <class PS, int LB, int NPR, int TA = 0>
struct Tc4Geom {
    static constexpr int P = PS::P;
    static constexpr int NKS = (P + 127 + 63) / 64;          // K steps of 64
    static constexpr int K = 64 * NKS;
    static constexpr int NT = (P + 127) / 128;                // output blocks (folded B, tcmul.cuh)
    static constexpr int NL = (NT + 1 + 7) / 8 * 8;           // B rows per digit (+ the fix row)
    static constexpr int PCOL = LB * NL;                      // D columns per product (multiple of 8)
    // N of the MMA: the products' rows packed (multiple of 8: one product of 8 rows -- the
    // up-sweep and u items -- no longer fetches 8 rows of zero padding per MMA)
    static constexpr int NB = (NPR * PCOL + 7) / 8 * 8;
    static constexpr int NBL = (NB + 15) / 16;                // 16-column TMEM loads in the epilogue
    // window rows: the descriptor starts at row 1 and reads rows up to 127 + 32*(2*NKS-1) + 32
    static constexpr int AROWS = 64 * NKS + 128;             // multiple of 8
    static constexpr int A_BYTES = AROWS * 16;
    static constexpr int HA_WORDS = AROWS / 8 + 8;           // 8 nibbles per word; nibble 128 + j = digit(a_j)
    static constexpr int HA_BYTES = (HA_WORDS * 4 + 127) / 128 * 128;
    // TA: 5 copies of hA, copy g shifted by g words (copy_g[x] = hA[x + g]) so that every lane's
    // window words start 16-byte aligned; copies 16 B apart modulo 128 (distinct bank groups)
    static constexpr int HA_COPIES = TA ? 5 : 1;
    static constexpr int HA_CSTRIDE = TA ? HA_BYTES + 16 : HA_BYTES;     // bytes between copies
    static constexpr int HA_TOTAL = (HA_COPIES * HA_CSTRIDE + 127) / 128 * 128;
    // Z (nibbles): bt reversed, Z[ZMARG + E - m] = digit(bt[m]), E = 128 NT - 1 (tcmul.cuh)
    static constexpr int PD = P % 8;
    static constexpr int R0 = (P - 1) % 32;                   // accumulator row of the fix row
    static constexpr int ZMARG = 128;
    static constexpr int ZB_END = ZMARG + 128 * NT;
    static constexpr int Z_NIB = (ZMARG + 128 * NT + P + 64 + 255) / 256 * 256;
    static constexpr int ZR_BYTES = Z_NIB / 2;
    static constexpr int NCHB = 2 * NKS;                      // 16-byte K-chunks per B row
    // B: K-chunk c of row r at 16-byte unit c (NB + 1) + r (one pad unit per chunk, so the B build's
    // stores of consecutive chunks land on distinct bank groups)
    static constexpr int BLD = NB + 1;                        // 16-byte units between K-chunks
    static constexpr int B_BYTES = NCHB * BLD * 16;
    static constexpr int SFCOL = NB;                          // scale-factor columns after the accumulators
    static constexpr int ACOL = NB + 8;                       // TA: A operand, 8 columns per K step
    static constexpr int NTA = TA ? ((TA - ACOL) / 8 < NKS ? (TA - ACOL) / 8 : NKS) : 0;
    static constexpr int TCOLS_USED = ACOL + 8 * NTA;
    static constexpr int TCOLS = TCOLS_USED <= 32 ? 32 : TCOLS_USED <= 64 ? 64 : TCOLS_USED <= 128 ? 128 : TCOLS_USED <= 256 ? 256 : 512;
    static constexpr int NCHK = PS::P8 / 8;
    static constexpr int CH = (NCHK + 1 + 127) / 128;
    static constexpr int OFF_A = 0;
    static constexpr int OFF_B = OFF_A + A_BYTES;
    static constexpr int OFF_HA = OFF_B + B_BYTES;
    static constexpr int OFF_ZR = OFF_HA + HA_TOTAL;
    static constexpr int OFF_BAR = OFF_ZR + NPR * LB * ZR_BYTES;
    static constexpr int SMEM = OFF_BAR + 128;
    // B build: one work item per Z unit u of each (pp, limb) group: it feeds chunk c = u - zrow(t)/32 of
    // every row t whose window covers it (each Z unit is read once, written to up to NT + 1 rows)
    static constexpr int ZFIX = (ZMARG + 128 * NT + 1 - 128 + R0 - P) / 32;   // fix row's first unit
    static constexpr int ZU0 = ZFIX < ZMARG / 32 ? ZFIX : ZMARG / 32;        // lowest unit read
    static constexpr int ZU1 = (ZMARG + 128 * (NT - 1)) / 32 + NCHB;       // one past the highest
    static constexpr int ZUN = ZU1 - ZU0;
    static constexpr int UITEMS = NPR * LB * ZUN;
    static constexpr int UPER = (UITEMS + 127) / 128;
    static_assert(NPR * PCOL <= NB && NB < BLD, "B build stores stay in B");
    static_assert(NB <= 256 && TCOLS_USED <= 512, "N too large");
    static_assert(!TA || (NTA >= 1 && 4 * (8 * NTA + 16) <= HA_BYTES), "TMEM A windows");
    static_assert(4 * (16 + NCHK) <= HA_BYTES, "hA too short (staging)");
    static_assert(4 * (AROWS / 8 + 5) <= HA_BYTES, "hA too short (windows)");
    static_assert(PD != 0 && NCHK * 8 > P, "p odd: the s-groups need the next chunk");
    static_assert(ZMARG + 128 * NT + 1 - 128 + R0 - P >= 0 && (1 + R0 - P) % 32 == 0, "fix row window");
    static_assert(ZMARG + 128 * (NT - 1) + K <= Z_NIB, "Z too short");
    static constexpr __host__ __device__ int zrow(int t) {     // nibble start of B row t's window
        return t < NT ? ZMARG + 128 * (NT - 1 - t) : ZMARG + 128 * NT + 1 - 128 + R0 - P;
    }
};

// idesc for kind::mxf4 (block-scaled layout): A = B = E2M1, scales UE8M0, K = 64, M = 128, N
__host__ __device__ constexpr uint32_t umma_idesc_mxf4(int N) {
    return (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(128 >> 4) << 24);
}

__device__ __forceinline__ void umma_mxf4(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate, uint32_t tsf) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(tsf), "r"(tsf));
}

__device__ __forceinline__ void umma_mxf4_w(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate, uint32_t tsf) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(tsf), "r"(tsf));
}

__device__ __forceinline__ void umma_mxf4_ta_w(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate, uint32_t tsf) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%5], [%6], p;\n\t}\n" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(tsf), "r"(tsf));
}

// A operand in TMEM ([a-tmem] form; scripts/probe/tmem_a_probe.cu)
__device__ __forceinline__ void umma_mxf4_ta(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate, uint32_t tsf) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%5], [%6], p;\n\t}\n" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(tsf), "r"(tsf));
}

// 8 B digits (reversed into one word: value i -> nibble 7 - i), digit l of each value
template <int LB>
__device__ __forceinline__ void digits_rev8(const int (&vals)[8], uint32_t (&dw)[LB]) {
#pragma unroll
    for (int l = 0; l < LB; l++) dw[l] = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        int v = vals[i];
#pragma unroll
        for (int l = 0; l < LB; l++) {
            int d = v;
            if (LB > 1) {
                const int qd = (v + 4 + 9 * 1024) / 9 - 1024;    // floor((v + 4) / 9)
                d = v - 9 * qd;
                v = qd;
            }
            dw[l] |= e2m1_code(d) << (4 * (7 - i));
        }
    }
}

// M = modulus; A = one digit (the small operand); LB digits for the B operand; NPR products per A.
// The B operand is folded (bt of tcmul.cuh): LB = 1 sums stay in {0, +-s, +-2s} (s = 1 or 3:
// e2m1-exact up to 6); LB > 1 sums are reduced mod M before their base-9 digits.
// RING (with TA > 0): every K step's A rows go through the TA-column TMEM window in rounds of
// NTA K steps (build rows -> tcgen05.st -> MMAs from TMEM -> wait -> next round); no A windows in
// shared memory at all, so the shared-memory traffic per item is only the B operand and staging.
// (an explicit minimum of 8 CTAs per SM, i.e. <= 64 registers, measured slower: 320 -> 310 M R/3
// products/s; note __launch_bounds__(128, 1) is NOT the same as (128): it let ptxas raise the
// R/3 kernels to 80 / 95 registers, 6 / 5 CTAs per SM, and the step lost 5%; session 4: the
// two-product kernel alone at (128, 8) -- 64 registers without spills instead of 72, 8 CTAs per SM
// instead of 7 -- made the keygen step 0.4% slower in three alternating rounds,
// profiles/r02s4/libab_tc4minb8.log)
template <class PS, int M, int LB, int NPR, bool XOPS = false, int TA = 0, bool RING = false>
__global__ void __launch_bounds__(128) tc4_mul_kernel(MulArgs a) {
    using G = Tc4Geom<PS, LB, NPR, TA>;
    static_assert(!RING || TA > 0, "RING streams A through TMEM");
    constexpr int P = PS::P;
    constexpr int CH = G::CH;
    constexpr int PD = G::PD;
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *sA = sm + G::OFF_A;
    uint8_t *sB = sm + G::OFF_B;
    uint32_t *sHA = reinterpret_cast<uint32_t *>(sm + G::OFF_HA);
    uint8_t *sZR = sm + G::OFF_ZR;
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + G::OFF_BAR);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sm + G::OFF_BAR + 64);
    const int tid = threadIdx.x, warp = tid >> 5;

    for (int i = tid; i < (G::OFF_BAR - G::OFF_B) / 16; i += 128)
        reinterpret_cast<uint4 *>(sB)[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    if (tid == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"((uint32_t)G::TCOLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    {   // scale factors: 8 columns of UE8M0 2^0 in every lane (SFA and SFB both read them)
        const uint32_t la = tmem + ((uint32_t)(warp * 32) << 16) + G::SFCOL;
        const uint32_t s = 0x7f7f7f7fu;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(la),
                     "r"(s), "r"(s), "r"(s), "r"(s), "r"(s), "r"(s), "r"(s), "r"(s));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    constexpr uint32_t IDESC = umma_idesc_mxf4(G::NB);
    uint32_t phase = 0;
    static_assert(G::zrow(G::NT) / 32 >= G::ZU0 && G::zrow(G::NT - 1) / 32 >= G::ZU0 &&
                  G::zrow(0) / 32 + G::NCHB == G::ZU1 && G::ZU1 * 16 <= G::ZR_BYTES, "B build units");

    uint4 pu[CH], pv[NPR][CH], pn[NPR][CH];
    int pa1 = 0, pb1[NPR];
#pragma unroll
    for (int pp = 0; pp < NPR; pp++) pb1[pp] = 0;
    // window rows 4m+s, s = (i + m/2) mod 4 (8 consecutive threads' 16-byte stores hit 8 distinct
    // bank groups), m = tid mod 128: nibble shifts are per-thread constants
    uint32_t wsh[4];
#pragma unroll
    for (int i = 0; i < 4; i++) wsh[i] = 16u * (uint32_t)(tid & 1) + 4u * (uint32_t)((i + (tid >> 1)) & 3);
    TcWork<NPR> wn;                                       // work item of the prefetched rows
    auto prefetch = [&](long long it) {
        if (it >= a.n_out) return;
        TcWork<NPR> &w = wn;
        tc_work<NPR>(a, it, w);
        const Opnd du = opnd_or_zero(w.du, w.unit_u);
#pragma unroll
        for (int h = 0; h < CH; h++) {
            const int c = tid + 128 * h;
            if (c < G::NCHK) pu[h] = load_chunk(du, c);
            const int cs = c == G::NCHK ? -1 : c;
#pragma unroll
            for (int pp = 0; pp < NPR; pp++) {
                const Opnd dv = opnd_or_zero(w.dv[pp], w.unit_v[pp] || (pp > 0 && w.orow[pp] < 0));
                if (c < G::NCHK) pv[pp][h] = load_chunk(dv, c);
                if (c <= G::NCHK && cs < G::NCHK - 1) pn[pp][h] = load_chunk(dv, cs + 1);
            }
        }
        if (tid == 0) {                                   // raw: decoded when staged (coef_fin)
            pa1 = load_raw(du, P - 1);
#pragma unroll
            for (int pp = 0; pp < NPR; pp++)
                pb1[pp] = load_raw(opnd_or_zero(w.dv[pp], w.unit_v[pp] || (pp > 0 && w.orow[pp] < 0)), P - 1);
        }
    };
    // ---- stage digits of work item w (registers -> hA / Z staging, which the MMAs do not read)
    auto stage = [&](const TcWork<NPR> &w, int (&fixab)[NPR]) {
#pragma unroll
        for (int pp = 0; pp < NPR; pp++) fixab[pp] = 0;
        if (tid == 0) {                                   // the prefetched raw scalars u[p-1], v[p-1]
            pa1 = coef_fin<XOPS>(w.du, w.unit_u, P - 1, pa1);
#pragma unroll
            for (int pp = 0; pp < NPR; pp++)
                pb1[pp] = (pp > 0 && w.orow[pp] < 0) ? 0 : coef_fin<XOPS>(w.dv[pp], w.unit_v[pp], P - 1, pb1[pp]);
        }
            // ---- stage digits: one 32-bit word (8 nibbles) per 8 coefficients
#pragma unroll
            for (int h = 0; h < CH; h++) {
                const int c = tid + 128 * h;
                if (c < G::NCHK) {
                    uint32_t word = 0;
                    if (w.du.bytes == 1 && !w.unit_u && !(XOPS && w.du.mod3)) {
                        word = e2m1_pack8_int8(pu[h].x, pu[h].y, w.du.scale);
                    } else {
                        int uv8[8];
                        decode_chunk(pu[h], w.du.bytes, w.du.scale, w.unit_u, c, uv8, XOPS ? w.du.mod3 : 0);
#pragma unroll
                        for (int i = 0; i < 8; i++) word |= e2m1_code(uv8[i]) << (4 * i);
                    }
                    SNTRUP_CHECK(4 * (16 + c + 1) <= G::HA_BYTES);
                    sHA[16 + c] = word;                                  // nibbles 128 + 8c + i
                    if constexpr (TA) {
#pragma unroll
                        for (int g = 1; g < G::HA_COPIES; g++) sHA[g * (G::HA_CSTRIDE / 4) + 16 + c - g] = word;
                    }
                }
                if (c <= G::NCHK) {
                    const int cs = c == G::NCHK ? -1 : c;
#pragma unroll
                    for (int pp = 0; pp < NPR; pp++) {
                        uint32_t *zr = reinterpret_cast<uint32_t *>(sZR + pp * LB * G::ZR_BYTES);
                        const bool fast = LB == 1 && w.dv[pp].bytes == 1 && !w.unit_v[pp] && !(XOPS && w.dv[pp].mod3);
                        const int zws = (G::ZB_END + (P - PD) - 8 - 8 * cs) / 8;    // s-group word
                        const int zwb = G::ZB_END / 8 - 1 - c;                      // b[8c+i]: nibble ZB_END-1-8c-i
                        SNTRUP_CHECK(cs >= G::NCHK - 1 || (8 * zws >= G::ZB_END && 8 * zws + 8 <= G::Z_NIB));
                        SNTRUP_CHECK(c >= G::NCHK || (zwb >= 0 && 8 * zwb + 8 <= G::ZB_END));
                        if (c == 0) fixab[pp] = pa1 * pb1[pp];
                        if (LB == 1 && fast) {
                            // SWAR: forward-packed chunks, s-group = pairwise sums of two shifted views
                            const int sc = w.dv[pp].scale;
                            const uint32_t W0 = c < G::NCHK ? e2m1_pack8_int8(pv[pp][h].x, pv[pp][h].y, sc) : 0u;
                            if (cs < G::NCHK - 1) {
                                const uint32_t W1 = e2m1_pack8_int8(pn[pp][h].x, pn[pp][h].y, sc);
                                zr[zws] = nibble_reverse(e2m1_pair_sum(__funnelshift_r(W0, W1, 4 * PD),
                                                                       __funnelshift_r(W0, W1, 4 * (PD - 1)), sc));
                            }
                            if (c < G::NCHK) {
                                uint32_t fw = W0;
                                if (c == 0)                                  // bt[0] = b[0] + b[p-1]
                                    fw = (W0 & ~0xFu) | e2m1_code(sc * (int)(int8_t)(pv[pp][h].x & 0xFFu) + pb1[pp]);
                                zr[zwb] = nibble_reverse(fw);
                            }
                            continue;
                        }
                        int vv8[8], vn8[8];
                        if (c < G::NCHK)
                            decode_chunk(pv[pp][h], w.dv[pp].bytes, w.dv[pp].scale, w.unit_v[pp], c, vv8,
                                         XOPS ? w.dv[pp].mod3 : 0);
                        else
#pragma unroll
                            for (int i = 0; i < 8; i++) vv8[i] = 0;
                        if (cs < G::NCHK - 1) {
                            // s-group: s[i] = b[i] + b[i-1], i = 8cs+PD+j, at nibble ZB_END + p - 1 - i
                            decode_chunk(pn[pp][h], w.dv[pp].bytes, w.dv[pp].scale, w.unit_v[pp], cs + 1, vn8,
                                         XOPS ? w.dv[pp].mod3 : 0);
                            int s8[8];
#pragma unroll
                            for (int j = 0; j < 8; j++) {
                                const int i0 = PD + j, i1 = PD + j - 1;
                                s8[j] = (i0 < 8 ? vv8[i0] : vn8[i0 - 8]) + (i1 < 8 ? vv8[i1] : vn8[i1 - 8]);
                                if (LB > 1) s8[j] = canon<M>(s8[j]);
                            }
                            uint32_t dw[LB];
                            digits_rev8<LB>(s8, dw);
#pragma unroll
                            for (int l = 0; l < LB; l++) zr[l * (G::ZR_BYTES / 4) + zws] = dw[l];
                        }
                        if (c < G::NCHK) {
                            uint32_t dw[LB];
                            if (c == 0) {
                                vv8[0] += pb1[pp];                       // bt[0] = b[0] + b[p-1]
                                if (LB > 1) vv8[0] = canon<M>(vv8[0]);
                            }
                            digits_rev8<LB>(vv8, dw);
#pragma unroll
                            for (int l = 0; l < LB; l++) zr[l * (G::ZR_BYTES / 4) + zwb] = dw[l];
                        }
                    }
                }
            }
    };

    // ES: the next item is staged while this item's MMAs run (its rows prefetched one iteration
    // earlier).  Not with two products per item: the second item's live state costs registers
    // (72 -> 86: 7 -> 5 CTAs per SM), measured slower in keygen.
    constexpr bool ES = NPR == 1;
    prefetch(blockIdx.x);
    TcWork<NPR> w = wn;
    int fixab[NPR];
    if (ES && blockIdx.x < a.n_out) {
        stage(w, fixab);
        prefetch(blockIdx.x + gridDim.x);
    }
#ifdef SNTRUP_WS_TRACE
    // phase timing (trace build): thread 0's clock between the loop's barriers, summed per CTA
    unsigned long long tph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tq = clock64();
#define TC4_PH(i) do { if (tid == 0) { const long long t_ = clock64(); tph[i] += t_ - tq; tq = t_; } } while (0)
#else
#define TC4_PH(i) do { } while (0)
#endif
    for (long long it = blockIdx.x; it < a.n_out; it += gridDim.x) {
        const long long nx = it + gridDim.x;
        if constexpr (!ES) {
            w = wn;
            stage(w, fixab);
        }
        TC4_PH(0);
        __syncthreads();
        TC4_PH(1);
        if constexpr (TA && !RING) {
            // ---- A rows into TMEM: lane r, K step ks = nibbles [1 + r + 64 ks, +64) of hA (the row the
            // shared-memory descriptor below starts at), 8 columns of 8 nibbles
            tc_fence_after();
            const int r1 = tid + 1, g = (r1 >> 3) - 4 * warp;             // 0..4
            const uint32_t sh = 4u * (uint32_t)(r1 & 7);
            const uint4 *src = reinterpret_cast<const uint4 *>(reinterpret_cast<const uint8_t *>(sHA) +
                                                               g * G::HA_CSTRIDE) + warp;
            const uint32_t la = tmem + ((uint32_t)(warp * 32) << 16) + G::ACOL;
            uint4 q0 = src[0];
#pragma unroll
            for (int ks = 0; ks < G::NTA; ks++) {
                const uint4 q1 = src[2 * ks + 1], q2 = src[2 * ks + 2];
                const uint32_t x[9] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w, q2.x};
                uint32_t o[8];
#pragma unroll
                for (int i = 0; i < 8; i++) o[i] = __funnelshift_r(x[i], x[i + 1], sh);
                asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(la + 8 * ks),
                             "r"(o[0]), "r"(o[1]), "r"(o[2]), "r"(o[3]), "r"(o[4]), "r"(o[5]), "r"(o[6]), "r"(o[7]));
                q0 = q2;
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        // ---- A windows: row rho = nibbles [rho, rho+32); rows 4m..4m+3 share word base m/2
#pragma unroll
        for (int kw = 0; kw < (RING ? 0 : (G::AROWS / 4 - 16 * G::NTA + 127) / 128); kw++) {
            const int m = 16 * G::NTA + tid + 128 * kw;          // rows >= 64 NTA: the K steps >= NTA
            if (m >= G::AROWS / 4) break;
            SNTRUP_CHECK(4 * ((m >> 1) + 5) <= G::HA_BYTES && 64 * (m + 1) <= G::A_BYTES);
            const uint32_t *src = sHA + (m >> 1);
            uint32_t wd[5];
#pragma unroll
            for (int i = 0; i < 5; i++) wd[i] = src[i];
            uint4 *dst = reinterpret_cast<uint4 *>(sA) + 4 * m;
#pragma unroll
            for (int i = 0; i < 4; i++) {
                uint4 o;
                o.x = __funnelshift_r(wd[0], wd[1], wsh[i]);
                o.y = __funnelshift_r(wd[1], wd[2], wsh[i]);
                o.z = __funnelshift_r(wd[2], wd[3], wsh[i]);
                o.w = __funnelshift_r(wd[3], wd[4], wsh[i]);
                dst[(i + (tid >> 1)) & 3] = o;
            }
        }
        // ---- B rows: each Z unit read once and stored into every row window that covers it
#pragma unroll
        for (int h = 0; h < G::UPER; h++) {
            const int w = tid + 128 * h;
            if (w >= G::UITEMS) break;
            const int pl = w / G::ZUN, u = G::ZU0 + (w - pl * G::ZUN);          // pl = pp * LB + l
            const int pp = pl / LB, l = pl - pp * LB;
            SNTRUP_CHECK(pl * (G::ZR_BYTES / 16) + u < NPR * LB * G::ZR_BYTES / 16);
            const uint4 z = reinterpret_cast<const uint4 *>(sZR)[pl * (G::ZR_BYTES / 16) + u];
            uint4 *dst = reinterpret_cast<uint4 *>(sB) + pp * G::PCOL + l * G::NL;
#pragma unroll
            for (int t = 0; t <= G::NT; t++) {
                const int c = u - G::zrow(t) / 32;
                if (c >= 0 && c < G::NCHB) {
                    // in range by construction (static_assert in Tc4Geom)
                    dst[c * G::BLD + t] = z;
                }
            }
        }
        fence_async_smem();
        if constexpr (RING) {
            // ---- A through the TMEM window in rounds of NTA K steps; the B rows above are built
            constexpr int NR = (G::NKS + G::NTA - 1) / G::NTA;
            const int r1 = tid + 1, g = (r1 >> 3) - 4 * warp;             // hA copy 0..4
            const uint32_t sh = 4u * (uint32_t)(r1 & 7);
            const uint4 *src = reinterpret_cast<const uint4 *>(reinterpret_cast<const uint8_t *>(sHA) +
                                                               g * G::HA_CSTRIDE) + warp;
            const uint32_t la = tmem + ((uint32_t)(warp * 32) << 16) + G::ACOL;
            const uint64_t bd0 = umma_desc(smem_u32(sB), G::BLD * 16, 128);
#pragma unroll 1
            for (int rr = 0; rr < NR; rr++) {
                if (rr > 0) {                                 // the window's previous MMAs are done
                    mbar_wait(bar, phase);
                    phase ^= 1;
                    tc_fence_after();
                }
                uint4 q0 = src[2 * G::NTA * rr];
#pragma unroll
                for (int kk = 0; kk < G::NTA; kk++) {
                    const int ks = G::NTA * rr + kk;
                    if (ks < G::NKS) {
                        const uint4 q1 = src[2 * ks + 1], q2 = src[2 * ks + 2];
                        const uint32_t x[9] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w, q2.x};
                        uint32_t o[8];
#pragma unroll
                        for (int i = 0; i < 8; i++) o[i] = __funnelshift_r(x[i], x[i + 1], sh);
                        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                                         la + 8 * kk),
                                     "r"(o[0]), "r"(o[1]), "r"(o[2]), "r"(o[3]), "r"(o[4]), "r"(o[5]), "r"(o[6]),
                                     "r"(o[7]));
                        q0 = q2;
                    }
                }
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                tc_fence_before();
                __syncthreads();
                if (warp == 0) {
                    tc_fence_after();
#pragma unroll
                    for (int kk = 0; kk < G::NTA; kk++) {
                        const int ks = G::NTA * rr + kk;
                        if (ks < G::NKS) {
                            const uint64_t bd = bd0 + (uint64_t)((ks * 32 * G::BLD) >> 4);
                            umma_mxf4_ta_w(tmem, tmem + G::ACOL + 8 * kk, bd, IDESC, ks > 0 ? 1u : 0u, tmem + G::SFCOL);
                        }
                    }
                    umma_commit_w(bar);
                }
            }
        } else {
        tc_fence_before();
        __syncthreads();
        if (warp == 0) {                                  // one elected lane of a converged warp
            tc_fence_after();
            const uint64_t bd0 = umma_desc(smem_u32(sB), G::BLD * 16, 128);
            const uint64_t ad0 = umma_desc(smem_u32(sA) + 16, 512, 128);
#pragma unroll
            for (int ks = 0; ks < G::NKS; ks++) {
                const uint64_t bd = bd0 + (uint64_t)((ks * 32 * G::BLD) >> 4);
                const uint64_t ad = ad0 + (uint64_t)((ks * 1024) >> 4);
                if (ks < G::NTA) umma_mxf4_ta_w(tmem, tmem + G::ACOL + 8 * ks, bd, IDESC, ks > 0 ? 1u : 0u, tmem + G::SFCOL);
                else umma_mxf4_w(tmem, ad, bd, IDESC, ks > 0 ? 1u : 0u, tmem + G::SFCOL);
            }
            umma_commit_w(bar);
        }
        }
        TC4_PH(2);
        const TcWork<NPR> nxt = wn;
        int fnx[NPR];
#pragma unroll
        for (int pp = 0; pp < NPR; pp++) fnx[pp] = 0;
        if constexpr (ES) {
            if (nx < a.n_out) {
                stage(nxt, fnx);
                TC4_PH(7);
                prefetch(nx + gridDim.x);
            }
        } else {
            prefetch(nx);
        }
        TC4_PH(3);
        if (tid == 0) mbar_wait(bar, phase);
        TC4_PH(4);
        phase ^= 1;
        __syncthreads();
        TC4_PH(5);
        tc_fence_after();
        // ---- epilogue: thread tid = TMEM lane = coefficient r of every block, straight to HBM
        const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
        int v[G::NBL][16];                                // every product's columns, one load
#pragma unroll
        for (int c16 = 0; c16 < G::NBL; c16++) {
            if (16 * c16 + 16 <= G::NB) tmem_ld16(lane_addr + 16 * c16, v[c16]);
            else tmem_ld8(lane_addr + 16 * c16, v[c16]);          // (columns 8..15 unused)
        }
        tmem_ld_wait();
#pragma unroll
        for (int pp = 0; pp < NPR; pp++) {
            auto comb = [&](int t) {
                int x = 0;
#pragma unroll
                for (int l = LB - 1; l >= 0; l--) {
                    const int col = pp * G::PCOL + l * G::NL + t;
                    x = 9 * x + __float2int_rn(__int_as_float(v[col >> 4][col & 15]));
                }
                return LB > 1 ? x % M : x;
            };
            int fix = 0;
            if (warp == 0) fix = __shfl_sync(FULL, comb(G::NT), G::R0);    // = D(p-1)
            const long long orow = w.orow[pp];
            if (orow < 0) continue;
            auto store = [&](auto *op) {
                constexpr int OSTRIDE = sizeof(*op) == 2 ? PS::P8 : PS::P16;
#pragma unroll
                for (int t = 0; t < G::NT; t++) {
                    const int k = 128 * t + tid;
                    if (k >= OSTRIDE) break;
                    int vv;
                    if (k == 0) vv = canon<M>(comb(0) - fix + fixab[pp] % M);
                    else if (M == 3 && LB == 1) {
                        const int col = pp * G::PCOL + t;
                        vv = (int)fmodc<3>(__int_as_float(v[col >> 4][col & 15]));   // exact: |D| < 2^20
                    }
                    else vv = canon<M>(comb(t));
                    if (k >= P) vv = 0;
                    if (XOPS && a.round3) vv -= canon<3>(vv);      // encapsulation's Round
                    op[k] = (std::remove_reference_t<decltype(*op)>)vv;
                }
            };
            uint8_t *orp = (pp == 1 && a.out2) ? (uint8_t *)a.out2 + orow * a.out2_stride * a.out_bytes
                                               : (uint8_t *)a.out + orow * a.out_stride * a.out_bytes;
            if (a.out_bytes == 2) store(reinterpret_cast<int16_t *>(orp));
            else store(reinterpret_cast<int8_t *>(orp));
        }
        tc_fence_before();
        TC4_PH(6);
        if constexpr (ES) {
            w = nxt;
#pragma unroll
            for (int pp = 0; pp < NPR; pp++) fixab[pp] = fnx[pp];
        }
    }
#ifdef SNTRUP_WS_TRACE
    if (tid == 0 && a.trace && TA == 0) {
        unsigned long long *tr = a.trace + (blockIdx.x % 160) * 16;
        for (int i = 0; i < 8; i++) atomicAdd(tr + 8 + i, tph[i]);
        atomicAdd(tr, (unsigned long long)((a.n_out - blockIdx.x + gridDim.x - 1) / gridDim.x));
    }
#endif
#undef TC4_PH
    tc_fence_before();
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)G::TCOLS));
}

}  // namespace sntrup
