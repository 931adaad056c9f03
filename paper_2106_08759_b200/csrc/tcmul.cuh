// tcmul.cuh -- batched ring products in R/q and R/3 on the 5th-generation tensor cores
// (tcgen05.mma kind::i8, int32 accumulators in TMEM).
//
// The ring product of section 3.3: full product c = a*b of two length-p
// polynomials, then reduction by x^p - x - 1 (x^p = x + 1), coefficients centered mod q (or 3).
// The paper computes it with Karatsuba / Schoenhage-Nussbaumer on 16-bit AVX2 lanes
// (P:4072-6339); on B200 the full product is a dense integer contraction, so it is posed as one
// GEMM per product on the int8 tensor cores:
//
//   raw[128 t + r] = sum_k A[r][k] * B[t][k],   A[r][k] = a[r + k - 127],  B[t][k] = b[128 t + 127 - k]
//
// (M = 128 output coefficients per block r, N = output blocks t, K = p + 127 rounded up to 32).
// A is a Hankel matrix.  In the no-swizzle K-major UMMA layout, core matrices are 8 rows x 16 B
// at SBO = 128 B (M direction) and LBO = 256 B (K direction); with those strides the tensor core
// reads element (r, k) of the descriptor's tile at byte 16*(r + k) + (k mod 16) of a "sliding
// window" buffer whose 16-byte row rho holds hA[rho .. rho+15] (hA = a shifted by 127).  So the
// whole 128 x K Hankel operand costs 16 B per row of a (16*(K+112) B) instead of 128*K B.
// B is materialised (N rows of K bytes) from aligned 16-byte chunks of the reversed b -- with the
// reduction x^p = x + 1 folded into it (TcGeom below), so the GEMM produces the reduced product
// directly: N = ceil(p/128) blocks (+ one fix row) and the epilogue stores straight to HBM.
//
// Coefficients of R/q do not fit int8: a big operand is split into limbs v = 64*hi + lo with
// lo in [-32, 31] and hi in [-62, 62] (|v| <= (q-1)/2 <= 3939; the folded B holds sums of two
// coefficients, |hi| <= 123).  A-limbs are separate MMAs into separate TMEM accumulators; B-limbs
// are stacked along N.  Small operands (R/3 elements, 3f, g, the unit) are one limb.  Exactness:
// every accumulator is an exact int32 sum (|sum| <= p * 62 * 123 < 2^24), combined mod q in the
// epilogue.
//
// One CTA (4 warps) per product, persistent over the grid; thread r owns TMEM lane r (output
// coefficient r of every block) in the epilogue.  Several CTAs per SM overlap one CTA's operand
// build / epilogue with another's MMAs.
#pragma once
#include <type_traits>

#include "common.cuh"
#include "ringmul.cuh"

namespace sntrup {

// ----------------------------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// UMMA shared-memory descriptor, SWIZZLE_NONE, K-major (version 1 for sm_100).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;                 // version
    return d;                               // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
}

// Instruction descriptor: kind::i8, D = s32, A = B = signed int8, both K-major, M = 128, N.
__host__ __device__ constexpr uint32_t umma_idesc_i8(int N, int M = 128) {
    return (2u << 4)                        // c_format S32
         | (1u << 7)                        // a_format signed int8
         | (1u << 10)                       // b_format signed int8
         | ((uint32_t)(N >> 3) << 17)       // n_dim
         | ((uint32_t)(M >> 4) << 24);      // m_dim
}

__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// Warp-collective forms (_w): the whole warp calls them converged and one elected lane issues.
// A tcgen05.mma issued by a lone thread of a diverged warp costs ~46 cycles of issue; from a
// converged warp through elect.sync the MMAs stream at the tensor core's own rate (16.9 cycles
// for M128 N32 K32 i8 = the 128 N / 256 floor; scripts/probe/mma_issue_probe.cu).
__device__ __forceinline__ void umma_i8_w(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit_w(uint64_t *bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
            smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    return ok != 0;
}

// Bounded wait: a descriptor or protocol bug must not hang the GPU (trap after ~2^31 cycles).
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    const long long t0 = clock64();
    while (!mbar_try_wait(bar, phase)) {
        if (clock64() - t0 > (1LL << 31)) __trap();
    }
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}
// 8 columns into v[0..7] (v[8..15] left untouched)
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, int (&v)[16]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ----------------------------------------------------------------------------------- geometry
// NPR products share one A operand per iteration (the down-sweep's two children share the
// parent's inverse): their B rows are stacked along N, so the A tile read by every MMA -- the
// dominant shared-memory traffic of a small-N GEMM -- is amortised over both products.
//
// Folded B operand.  The reduction x^p = x + 1 is folded into B: with the Laurent extension
//   bt[m] = b[m] (m >= 1),  bt[0] = b[0] + b[p-1],  bt[m] = b[m+p] + b[m+p-1] (-p < m < 0),
// the Toeplitz sum  sum_j a[j] bt[k - j]  equals the reduced product coefficient c[k] for every
// 1 <= k < p (the wrapped terms raw[k+p] and raw[k+p-1] of section 3.3's reduction), and
// c[0] + raw[p-1] for k = 0.  So the GEMM only needs the NT = ceil(p/MM) output blocks of the
// reduced product (half the N of the full product, no fold pass), and c[0] is fixed with
// c[0] = D(0) - D(p-1) + a[p-1] b[p-1] (raw[p-1] = c[p-1] - a[p-1] b[p-1]).  An extra B row
// ("fix row") repeats output p-1 in accumulator row R0 = (p-1) mod 16, a lane of warp 0, so
// thread 0 gets it with one shuffle.
//   Z (per B limb) holds bt reversed: Z[ZMARG + E - m] = limb(bt[m]), E = MM*NT - 1; B row t
//   (t < NT) is the window Z[ZMARG + MM(NT-1-t) + k], the fix row Z[ZMARG + MM NT + 1 - MM + R0 - p + k].
template <class PS, int LA, int LB, int NPR, int MM = 128>
struct TcGeom {
    static_assert(MM == 64 || MM == 128, "M is 64 or 128");
    static constexpr int P = PS::P;
    static constexpr int NKS = (P + MM - 1 + 31) / 32;       // K steps of 32
    static constexpr int K = 32 * NKS;
    static constexpr int NT = (P + MM - 1) / MM;              // output blocks of MM coefficients
    // the fix row costs nothing when NT + 1 rows still fit the 8-row padding; otherwise (NT a
    // multiple of 8: 953, 1013) c[p-1] goes from its own lane to thread 0 through shared memory
    static constexpr bool FIXROW = (NT + 1 + 7) / 8 == (NT + 7) / 8;
    static constexpr int NROWS = NT + (FIXROW ? 1 : 0);       // B rows built per limb
    static constexpr int NL = (NROWS + 7) / 8 * 8;            // B rows per limb (padded)
    static constexpr int PCOL = (LB * NL + 15) / 16 * 16;    // B rows (= D columns) per product
    static constexpr int NB = NPR * PCOL;                    // N of the MMA
    static constexpr int AROWS = 32 * NKS + MM - 15;         // window rows 0..AROWS-1 (row 0 unused)
    static constexpr int A_BYTES = (AROWS + 7) / 8 * 128;    // 16 B per row, 128-aligned
    static constexpr int AROWS4 = (AROWS + 3) / 4;            // window rows are built 4 at a time
    static constexpr int HA_LEN = (4 * AROWS4 + 20 + 127) / 128 * 128;   // hA[MM + j] = limb(a_j)
    static constexpr int PD = P % 8;                          // s-groups start at 8c + PD
    static constexpr int R0 = (P - 1) % 16;                   // accumulator row of the fix row
    static constexpr int ZMARG = MM;
    static constexpr int Z_LEN = (ZMARG + MM * NT + P + 32 + 127) / 128 * 128;
    static constexpr int ZB_END = ZMARG + MM * NT;            // b part below, s part from here
    // B: K-chunk c of row r at 16-byte unit c (NB + 1) + r (one pad unit per chunk, so the B
    // build's stores of consecutive chunks land on distinct bank groups)
    static constexpr int BLD = NB + 1;
    static constexpr int B_BYTES = 2 * NKS * BLD * 16;
    static constexpr int TCOLS_USED = LA * NB;
    static constexpr int TCOLS = TCOLS_USED <= 32 ? 32 : TCOLS_USED <= 64 ? 64 : TCOLS_USED <= 128 ? 128 : 256;
    static constexpr int NCHK = PS::P8 / 8;                   // 8-coefficient input chunks
    static constexpr int CH = (NCHK + 1 + 127) / 128;         // chunks per thread (+ the s-group -1)
    // smem carve-up (bytes, all 128-aligned)
    static constexpr int OFF_A = 0;
    static constexpr int OFF_B = OFF_A + LA * A_BYTES;
    static constexpr int OFF_HA = OFF_B + B_BYTES;
    static constexpr int OFF_ZR = OFF_HA + LA * HA_LEN;
    static constexpr int OFF_BAR = OFF_ZR + NPR * LB * Z_LEN;
    static constexpr int SMEM = OFF_BAR + 128;
    // resident CTAs the shared memory allows (up to 4): register budget for __launch_bounds__
    static constexpr int MINB = (227 * 1024) / (SMEM + 1024) < 4 ? (227 * 1024) / (SMEM + 1024) : 4;
    static_assert(NB <= 256, "N too large");
    static_assert(MM + PS::P8 <= HA_LEN, "hA too short");
    static_assert(4 * AROWS4 * 16 <= A_BYTES, "A region too short");
    static_assert(PD != 0 && NCHK * 8 > P, "p odd: the s-groups need the next chunk");
    static_assert(ZMARG + MM * NT + 1 - MM + R0 - P >= 0 && (1 + R0 - P) % 16 == 0, "fix row window");
    static_assert(ZMARG + MM * (NT - 1) + K <= Z_LEN, "Z too short");
    static constexpr int NCHB = 2 * NKS;                      // 16-byte K-chunks per B row
    // start (bytes) of B row t's window in Z
    static constexpr __host__ __device__ int zrow(int t) {
        return t < NT ? ZMARG + MM * (NT - 1 - t) : ZMARG + MM * NT + 1 - MM + R0 - P;
    }
    // B build: one work item per 16-byte Z unit u of each (pp, limb) group; it feeds chunk
    // c = u - zrow(t)/16 of every row t whose window covers it (each Z unit read once)
    static constexpr int ZU0 = (FIXROW && zrow(NT) / 16 < ZMARG / 16) ? zrow(NT) / 16 : ZMARG / 16;
    static constexpr int ZU1 = zrow(0) / 16 + NCHB;
    static constexpr int ZUN = ZU1 - ZU0;
    static constexpr int UITEMS = NPR * LB * ZUN;
    static_assert(ZU1 * 16 <= Z_LEN, "B build units");
    static_assert(NPR * PCOL <= NB && NB < BLD && NCHB * BLD * 16 == B_BYTES, "B build stores stay in B");
};

// limb l (0 = hi, 1 = lo) of a centered coefficient when the operand has L limbs
template <int L>
__device__ __forceinline__ int limb_of(int v, int l) {
    if (L == 1) return v;
    const int lo = ((v + 32) & 63) - 32;
    return l == 0 ? (v - lo) >> 6 : lo;
}

// One operand row of a work item: its first byte, element size, load scale and mod-3 pre-op.
struct Opnd {
    const uint8_t *row;
    int bytes, scale, mod3;
};

__device__ __forceinline__ Opnd opnd(const RowDesc &d, long long r) {
    Opnd o;
    o.row = (const uint8_t *)d.ptr + r * d.stride * d.bytes;
    o.bytes = d.bytes; o.scale = d.scale; o.mod3 = d.mod3;
    return o;
}

// 16 raw bytes of chunk c (coefficients 8c .. 8c+7) of an operand row (int16: 16 B, int8: 8 B)
__device__ __forceinline__ uint4 load_chunk(const Opnd &d, int c) {
    if (d.bytes == 2) return __ldg(reinterpret_cast<const uint4 *>(d.row) + c);
    const uint2 v = __ldg(reinterpret_cast<const uint2 *>(d.row) + c);
    return make_uint4(v.x, v.y, 0, 0);
}

// Prefetch without waiting: the prefetches issue loads whose results are consumed an iteration
// later, so nothing in them may depend on a loaded value.  An absent or unit operand (whose data
// the decode ignores) loads from this zero row instead of selecting a zero VALUE after the load
// (a select on the value made every prefetch wait for global-memory latency: 2.5k of 5.4k cycles
// per fp4 item, scripts/tc4_phase_trace.py); the scalar coefficient is loaded raw and decoded
// (unit, scale, mod-3) when staged.
__device__ uint4 g_zero_rows[192];                       // 3 KB >= the longest row (1280 x int16)
__device__ __forceinline__ Opnd opnd_or_zero(const Opnd &d, bool none) {
    Opnd o = d;
    o.row = none ? reinterpret_cast<const uint8_t *>(g_zero_rows) : d.row;
    return o;
}
__device__ __forceinline__ int load_raw(const Opnd &d, int k) {
    return d.bytes == 1 ? (int)((const int8_t *)d.row)[k] : (int)((const int16_t *)d.row)[k];
}
template <bool XOPS>
__device__ __forceinline__ int coef_fin(const Opnd &d, bool unit, int k, int raw) {
    if (unit) return k == 0 ? 1 : 0;
    const int v = raw * d.scale;
    return (XOPS && d.mod3) ? canon<3>(v) : v;
}

// coefficient k of an operand row (decoded: scale, optional mod-3 pre-op)
template <bool XOPS>
__device__ __forceinline__ int opnd_coef(const Opnd &d, bool unit, int k) {
    if (unit) return k == 0 ? 1 : 0;
    int v = d.bytes == 1 ? (int)((const int8_t *)d.row)[k] : (int)((const int16_t *)d.row)[k];
    v *= d.scale;
    return (XOPS && d.mod3) ? canon<3>(v) : v;
}

__device__ __forceinline__ void decode_chunk(const uint4 r, int bytes, int scale, bool unit, int c, int (&v)[8],
                                             int mod3 = 0) {
    if (bytes == 2) {
        const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
        for (int i = 0; i < 8; i++) v[i] = scale * (int)(int16_t)(w[i >> 1] >> (16 * (i & 1)));
    } else {
        const uint32_t w[2] = {r.x, r.y};
#pragma unroll
        for (int i = 0; i < 8; i++) v[i] = scale * (int)(int8_t)(w[i >> 2] >> (8 * (i & 3)));
    }
    if (mod3) {
#pragma unroll
        for (int i = 0; i < 8; i++) v[i] = canon<3>(v[i]);
    }
    if (unit) {
#pragma unroll
        for (int i = 0; i < 8; i++) v[i] = (c == 0 && i == 0) ? 1 : 0;
    }
}

__device__ __forceinline__ uint32_t pack4(int a, int b, int c, int d) {
    return (uint32_t)(a & 0xff) | ((uint32_t)(b & 0xff) << 8) | ((uint32_t)(c & 0xff) << 16) |
           ((uint32_t)(d & 0xff) << 24);
}

// Operands of work item `it`: u -> A role; v[pp] -> B role of product pp, written to out row
// orow[pp] (orow < 0: no such product).
template <int NPR>
struct TcWork {
    Opnd du; bool unit_u;
    Opnd dv[NPR]; bool unit_v[NPR];
    long long orow[NPR];
};

template <int NPR>
__device__ __forceinline__ void tc_work(const MulArgs &a, long long it, TcWork<NPR> &w) {
    w.unit_u = false;
#pragma unroll
    for (int pp = 0; pp < NPR; pp++) { w.unit_v[pp] = false; w.orow[pp] = -1; w.dv[pp] = opnd(a.X, 0); }
    if constexpr (NPR == 2) {
        if (a.mode == MUL_UP0) {
            const long long i1 = 2 * it + 1;
            w.unit_u = i1 >= a.cnt_in;
            w.du = opnd(a.Y, w.unit_u ? 0 : i1);
            w.dv[0] = opnd(a.X, 2 * it); w.orow[0] = 2 * it;
            w.dv[1] = opnd(a.Y, 2 * it); w.orow[1] = it;          // into out2
            return;
        }
        // MUL_DOWN2: parent it; out[2it] = Y[it] * X[2it+1] (unit if absent), out[2it+1] = Y[it] * X[2it]
        // MUL_DOWNH2: parent it; out[2it] = Y[it] * X[2it], out[2it+1] = Y[it] * X[2it+1] (if present)
        const bool noswap = a.mode == MUL_DOWNH2;
        w.du = opnd(a.Y, it);
        w.dv[0] = opnd(a.X, noswap ? 2 * it : 2 * it + 1);
        w.unit_v[0] = !noswap && 2 * it + 1 >= a.cnt_in; w.orow[0] = 2 * it;
        w.dv[1] = opnd(a.X, noswap ? 2 * it + 1 : 2 * it);
        w.orow[1] = (2 * it + 1 < a.cnt_in) ? 2 * it + 1 : -1;
    } else {
        RowDesc du, dv; long long ru, rv; bool uv = false, uu = false;
        if (a.mode == MUL_ZIP) {
            du = a.X; ru = it; dv = a.Y; rv = it;
        } else if (a.mode == MUL_PAIRS) {
            du = a.X; ru = 2 * it; dv = a.X; rv = 2 * it + 1;
            uv = rv >= a.cnt_in;
        } else if (a.mode == MUL_SIB) {
            du = a.X; ru = it; dv = a.Y; rv = it ^ 1;
            uv = rv >= a.cnt_in;
        } else if (a.mode == MUL_ODDSIB) {
            du = a.Y; ru = 2 * it; dv = a.X; rv = 2 * it + 1;
        } else if (a.mode == MUL_DOWNH) {
            du = a.Y; ru = it >> 1; dv = a.X; rv = it;
        } else {
            du = a.Y; ru = it >> 1; dv = a.X; rv = it ^ 1;
            uv = rv >= a.cnt_in;
        }
        if (a.swap) {
            const RowDesc td = du; du = dv; dv = td;
            const long long tr = ru; ru = rv; rv = tr;
            uu = uv; uv = false;
        }
        w.du = opnd(du, ru); w.unit_u = uu;
        w.dv[0] = opnd(dv, rv); w.unit_v[0] = uv; w.orow[0] = a.mode == MUL_ODDSIB ? 2 * it + 1 : it;
    }
}

// M = modulus (3 or q); LA / LB = limbs of the A-role / B-role operand; NPR products per A;
// MM = MMA M (output coefficients per block).  With MM = 64 each MMA reads half the A bytes and
// the accumulator row r lives in TMEM lane 32(r/16) + r%16 (probed: scripts/probe/tmem_m64_probe.cu).
// XOPS: honour the operand pre-op (RowDesc.mod3) and the output post-op (MulArgs.round3) of the
// KEM core; compiled out of the keygen instantiations.
// NT threads per CTA and ST operand stages: ST = 1 (NT = 128) is the plain loop -- several CTAs
// per SM overlap one CTA's operand build with another's MMAs; ST = 2 (NT = 256, one or two CTAs
// per SM) software-pipelines inside the CTA: item k+1's operands are built in the second stage and
// its MMAs issued before item k's epilogue, which then overlaps them.
// NH > 1 (big x big, ST = 1): the K range is processed in NH parts through operand buffers sized
// for one part (A windows and B rows of KH = ceil(NKS / NH) K steps; each part's MMAs accumulate
// into the same TMEM columns and are waited for before the next part is built), which cuts the
// shared memory per CTA from 72 KB to 43 KB (NH = 2, two products per item) -- more resident CTAs
// per SM, at the same per-item chain length.
template <class G, int LA, int LB, int NPR, int MM, int NH>
struct TcParts {
    static constexpr int KH = (G::NKS + NH - 1) / NH;         // K steps per part
    static constexpr int AROWS = 32 * KH + MM - 15;
    static constexpr int A_BYTES = NH == 1 ? G::A_BYTES : (AROWS + 7) / 8 * 128;
    static constexpr int AROWS4 = NH == 1 ? G::AROWS4 : (AROWS + 3) / 4;
    static constexpr int B_BYTES = NH == 1 ? G::B_BYTES : 2 * KH * G::BLD * 16;
    static constexpr int ZUN = G::ZUN - G::NCHB + 2 * KH;    // Z units feeding one part's chunks
    static constexpr int UITEMS = NPR * LB * ZUN;
    static constexpr int SMEM = LA * A_BYTES + B_BYTES + LA * G::HA_LEN + NPR * LB * G::Z_LEN + 128;
    static constexpr int BY_SMEM = (227 * 1024) / (SMEM + 1024);
    static constexpr int CAPB = NH == 2 && NPR == 2 ? 5 : 6;  // register cap: 65536 / (128 CAPB) per thread
    static constexpr int MINB = NH == 1 ? G::MINB : (BY_SMEM < CAPB ? BY_SMEM : CAPB);
    static_assert(4 * AROWS4 * 16 <= A_BYTES, "A part too short");
    // (the build skips window rows past the whole operand's AROWS4 groups, so its hA reads stay
    // inside HA_LEN also when NKS is not a multiple of NH)
};

template <class PS, int M, int LA, int LB, int NPR, int MM = 128, bool XOPS = false, int NT = 128, int ST = 1, int NH = 1>
__global__ void __launch_bounds__(NT, (ST == 1 ? TcParts<TcGeom<PS, LA, LB, NPR, MM>, LA, LB, NPR, MM, NH>::MINB : 1))
tc_mul_kernel(MulArgs a) {
    using G = TcGeom<PS, LA, LB, NPR, MM>;
    using H = TcParts<G, LA, LB, NPR, MM, NH>;
    static_assert(ST == 1 || (ST == 2 && MM == 128 && NT == 256), "pipelined variant: M = 128, 8 warps");
    static_assert(ST == 2 || NT == 128, "plain variant: 4 warps");
    static_assert(NH == 1 || (ST == 1 && LA == 2 && LB == 2), "K parts: the big x big plain variant");
    constexpr int P = PS::P;
    constexpr int PD = G::PD;
    constexpr int CH = (G::NCHK + 1 + NT - 1) / NT;           // staging chunks per thread (+ s-group -1)
    constexpr int UPER = (H::UITEMS + NT - 1) / NT;
    constexpr int ASTG = LA * H::A_BYTES;                     // one stage's A windows
    constexpr int OFF_B = ST * ASTG;                          // B of stage b at OFF_B + b B_BYTES
    constexpr int OFF_HA = OFF_B + ST * H::B_BYTES;
    constexpr int OFF_ZR = OFF_HA + LA * G::HA_LEN;
    constexpr int OFF_BAR = OFF_ZR + NPR * LB * G::Z_LEN;
    constexpr int TCU = ST * LA * G::NB;                      // accumulators of every stage
    constexpr int TCOLS = TCU <= 32 ? 32 : TCU <= 64 ? 64 : TCU <= 128 ? 128 : 256;
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *sHA = sm + OFF_HA;
    uint8_t *sZR = sm + OFF_ZR;
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + OFF_BAR);          // bar[b], one per stage
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sm + OFF_BAR + 64);
    int *fixs = reinterpret_cast<int *>(sm + OFF_BAR + 72);     // c[p-1] hand-off (no fix row), per product
    int *fixab_s = reinterpret_cast<int *>(sm + OFF_BAR + 88);  // a[p-1] b[p-1] per stage and product
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    static_assert(88 + 4 * ST * NPR <= 128, "barrier area");

    // ---- one-time setup: zero staging + B (pads stay zero forever), barriers, TMEM
    for (int i = tid; i < (OFF_BAR - OFF_B) / 16; i += NT)
        reinterpret_cast<uint4 *>(sm + OFF_B)[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    if (tid == 0) {
#pragma unroll
        for (int b = 0; b < ST; b++) mbar_init(bar + b, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"((uint32_t)TCOLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    constexpr uint32_t IDESC = umma_idesc_i8(G::NB, MM);
    uint32_t phases = 0;                                    // mbarrier parity, bit b = stage b

    // register prefetch of the next work item's rows (in flight during the MMAs / epilogue):
    // chunk c of u and of every v, chunk c+1 of v (the s-groups straddle chunks), and for
    // thread 0 the scalars u[p-1], v[p-1] (bt[0] and the c[0] fix)
    uint4 pu[CH], pv[NPR][CH], pn[NPR][CH];
    int pa1 = 0, pb1[NPR];
#pragma unroll
    for (int pp = 0; pp < NPR; pp++) pb1[pp] = 0;
    // A-window rows 4m+s, s = (i + m/2) mod 4: 8 consecutive threads' 16-byte stores then hit 8
    // distinct bank groups (64m + 16s); m = tid mod NT, so the byte selectors are per-thread
    // constants
    uint32_t wsel[4];
#pragma unroll
    for (int i = 0; i < 4; i++) wsel[i] = 0x3210u + (uint32_t)((i + (tid >> 1)) & 3) * 0x1111u;   // bytes s..s+3
    TcWork<NPR> wn;                                       // work item of the prefetched rows
    auto prefetch = [&](long long it) {
        if (it >= a.n_out) return;
        TcWork<NPR> &w = wn;
        tc_work<NPR>(a, it, w);
        const Opnd du = opnd_or_zero(w.du, w.unit_u);
#pragma unroll
        for (int h = 0; h < CH; h++) {
            const int c = tid + NT * h;
            if (c < G::NCHK) pu[h] = load_chunk(du, c);
            const int cs = c == G::NCHK ? -1 : c;                // thread NCHK: s-group -1
#pragma unroll
            for (int pp = 0; pp < NPR; pp++) {
                const Opnd dv = opnd_or_zero(w.dv[pp], w.unit_v[pp] || (pp > 0 && w.orow[pp] < 0));
                if (c < G::NCHK) pv[pp][h] = load_chunk(dv, c);
                if (c <= G::NCHK && cs < G::NCHK - 1) pn[pp][h] = load_chunk(dv, cs + 1);
            }
        }
        if (tid == 0) {                                       // raw: decoded when staged (coef_fin)
            pa1 = load_raw(du, P - 1);
#pragma unroll
            for (int pp = 0; pp < NPR; pp++)
                pb1[pp] = load_raw(opnd_or_zero(w.dv[pp], w.unit_v[pp] || (pp > 0 && w.orow[pp] < 0)), P - 1);
        }
    };

    // ---- stage limbs of the prefetched item (8-byte aligned groups): hA_l[MM + j] = limb_l(u_j);
    //      Z_{pp,l}: b part (chunk c reversed) and s part (s-group c: bt at 8c+PD .. 8c+PD+7)
    auto stage = [&](const TcWork<NPR> &w, int (&fixab)[NPR], int b) {
#pragma unroll
        for (int pp = 0; pp < NPR; pp++) fixab[pp] = 0;
        if (tid == 0) {                                       // the prefetched raw scalars u[p-1], v[p-1]
            pa1 = coef_fin<XOPS>(w.du, w.unit_u, P - 1, pa1);
#pragma unroll
            for (int pp = 0; pp < NPR; pp++)
                pb1[pp] = (pp > 0 && w.orow[pp] < 0) ? 0 : coef_fin<XOPS>(w.dv[pp], w.unit_v[pp], P - 1, pb1[pp]);
        }
#pragma unroll
        for (int h = 0; h < CH; h++) {
            const int c = tid + NT * h;
            if (c < G::NCHK) {
                int uv8[8];
                decode_chunk(pu[h], w.du.bytes, w.du.scale, w.unit_u, c, uv8, XOPS ? w.du.mod3 : 0);
#pragma unroll
                for (int l = 0; l < LA; l++) {
                    int x[8];
#pragma unroll
                    for (int i = 0; i < 8; i++) x[i] = limb_of<LA>(uv8[i], l);
                    SNTRUP_CHECK(MM + 8 * c + 8 <= G::HA_LEN);
                    *reinterpret_cast<uint2 *>(sHA + l * G::HA_LEN + MM + 8 * c) =
                        make_uint2(pack4(x[0], x[1], x[2], x[3]), pack4(x[4], x[5], x[6], x[7]));
                }
            }
            if (c <= G::NCHK) {
                const int cs = c == G::NCHK ? -1 : c;               // s-group index
#pragma unroll
                for (int pp = 0; pp < NPR; pp++) {
                    int vv8[8], vn8[8];
                    if (c < G::NCHK)
                        decode_chunk(pv[pp][h], w.dv[pp].bytes, w.dv[pp].scale, w.unit_v[pp], c, vv8,
                                     XOPS ? w.dv[pp].mod3 : 0);
                    else
#pragma unroll
                        for (int i = 0; i < 8; i++) vv8[i] = 0;
                    const bool has_s = cs < G::NCHK - 1;
                    if (has_s)
                        decode_chunk(pn[pp][h], w.dv[pp].bytes, w.dv[pp].scale, w.unit_v[pp], cs + 1, vn8,
                                     XOPS ? w.dv[pp].mod3 : 0);
                    uint8_t *zr = sZR + pp * LB * G::Z_LEN;
                    if (has_s) {
                        // s[i] = b[i] + b[i-1] for i = 8cs+PD+j, j = 0..7, at Z[ZB_END + p - 1 - i]
                        int s8[8];
#pragma unroll
                        for (int j = 0; j < 8; j++) {
                            const int i0 = PD + j, i1 = PD + j - 1;
                            s8[j] = (i0 < 8 ? vv8[i0] : vn8[i0 - 8]) + (i1 < 8 ? vv8[i1] : vn8[i1 - 8]);
                        }
                        const int zo = G::ZB_END + (P - PD) - 8 - 8 * cs;
                        SNTRUP_CHECK(zo >= G::ZB_END && zo + 8 <= G::Z_LEN && (zo & 7) == 0);
#pragma unroll
                        for (int l = 0; l < LB; l++) {
                            int x[8];
#pragma unroll
                            for (int j = 0; j < 8; j++) x[j] = limb_of<LB>(s8[j], l);
                            *reinterpret_cast<uint2 *>(zr + l * G::Z_LEN + zo) =
                                make_uint2(pack4(x[7], x[6], x[5], x[4]), pack4(x[3], x[2], x[1], x[0]));
                        }
                    }
                    if (c < G::NCHK) {
                        if (c == 0) {
                            vv8[0] += pb1[pp];                     // bt[0] = b[0] + b[p-1]
                            fixab[pp] = pa1 * pb1[pp];
                            if (NT == 256) fixab_s[b * NPR + pp] = fixab[pp];   // for the other warp group
                        }
                        const int zo = G::ZB_END - 8 - 8 * c;      // b[8c+i] at ZB_END - 1 - 8c - i
                        SNTRUP_CHECK(zo >= 0 && zo + 8 <= G::ZB_END);
#pragma unroll
                        for (int l = 0; l < LB; l++) {
                            int x[8];
#pragma unroll
                            for (int i = 0; i < 8; i++) x[i] = limb_of<LB>(vv8[i], l);
                            *reinterpret_cast<uint2 *>(zr + l * G::Z_LEN + zo) =
                                make_uint2(pack4(x[7], x[6], x[5], x[4]), pack4(x[3], x[2], x[1], x[0]));
                        }
                    }
                }
            }
        }
    };

    // ---- operands of stage b: A sliding windows (row rho = hA[rho .. rho+15], the descriptor
    //      starts at row 1; each work item builds rows 4m .. 4m+3 from 5 words) and B rows
    //      (row pp*PCOL + l*NL + t, K-chunk c = 16-byte unit c of the row's Z window)
    auto build = [&](int b, int h = 0) {
        uint8_t *sA = sm + b * ASTG;
        uint8_t *sB = sm + OFF_B + b * H::B_BYTES;
#pragma unroll
        for (int l = 0; l < LA; l++) {
#pragma unroll
            for (int kw = 0; kw < (H::AROWS4 + NT - 1) / NT; kw++) {
                const int m = tid + NT * kw;
                if (m >= H::AROWS4) break;
                const int mg = m + 8 * H::KH * h;               // window rows 4 mg .. of the whole operand
                if (NH > 1 && mg >= G::AROWS4) break;           // last part of an odd NKS: rows no MMA reads
                SNTRUP_CHECK(4 * (mg + 5) <= G::HA_LEN && 64 * (m + 1) <= H::A_BYTES);
                const uint32_t *src = reinterpret_cast<const uint32_t *>(sHA + l * G::HA_LEN) + mg;
                uint32_t wd[5];
#pragma unroll
                for (int i = 0; i < 5; i++) wd[i] = src[i];
                uint4 *dst = reinterpret_cast<uint4 *>(sA + l * H::A_BYTES) + 4 * m;
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    uint4 o;
                    o.x = __byte_perm(wd[0], wd[1], wsel[i]);
                    o.y = __byte_perm(wd[1], wd[2], wsel[i]);
                    o.z = __byte_perm(wd[2], wd[3], wsel[i]);
                    o.w = __byte_perm(wd[3], wd[4], wsel[i]);
                    dst[(i + (tid >> 1)) & 3] = o;
                }
            }
        }
        // each Z unit read once and stored into every row window that covers it (part h: the
        // chunks 2 KH h .. of every row)
        const int c0 = 2 * H::KH * h;
#pragma unroll
        for (int hh = 0; hh < UPER; hh++) {
            const int w = tid + NT * hh;
            if (w >= H::UITEMS) break;
            const int pl = w / H::ZUN, u = G::ZU0 + c0 + (w - pl * H::ZUN);     // pl = pp * LB + l
            const int pp = pl / LB, l = pl - pp * LB;
            if (NH > 1 && u >= G::ZU1) continue;
            SNTRUP_CHECK(pl * (G::Z_LEN / 16) + u < NPR * LB * G::Z_LEN / 16);
            const uint4 z = reinterpret_cast<const uint4 *>(sZR)[pl * (G::Z_LEN / 16) + u];
            uint4 *dst = reinterpret_cast<uint4 *>(sB) + pp * G::PCOL + l * G::NL;
#pragma unroll
            for (int t = 0; t < G::NROWS; t++) {
                const int c = u - G::zrow(t) / 16;
                const int cl = c - c0;
                if (cl >= 0 && cl < 2 * H::KH && c < G::NCHB) {
                    // in range by construction: base + t < NPR PCOL <= NB < BLD and cl < 2 KH
                    dst[cl * G::BLD + t] = z;
                }
            }
        }
        fence_async_smem();
    };

    // ---- MMAs of stage b (warp 0, one elected lane) into accumulator set b; descriptors advance by adding to
    //      the start-address field
    auto issue = [&](int b, int h = 0) {
        tc_fence_after();
        const uint64_t bd0 = umma_desc(smem_u32(sm + OFF_B + b * H::B_BYTES), G::BLD * 16, 128);
        const uint64_t ad0 = umma_desc(smem_u32(sm + b * ASTG) + 16, 256, 128);
        const uint32_t acc = tmem + (uint32_t)(b * LA * G::NB);
        const int ksn = (G::NKS - h * H::KH) < H::KH ? (G::NKS - h * H::KH) : H::KH;
#pragma unroll 1
        for (int ks = 0; ks < ksn; ks++) {
            const uint64_t bd = bd0 + (uint64_t)((ks * 32 * G::BLD) >> 4);
#pragma unroll
            for (int l = 0; l < LA; l++) {
                const uint64_t ad = ad0 + (uint64_t)((l * H::A_BYTES + ks * 512) >> 4);
                umma_i8_w(acc + l * G::NB, ad, bd, IDESC, (ks > 0 || h > 0) ? 1u : 0u);
            }
        }
        umma_commit_w(bar + b);
    };

    // ---- epilogue of accumulator set b: thread = TMEM lane = coefficient r of every block;
    //      outputs go straight to HBM (lane-consecutive coefficients: coalesced).  With 8 warps
    //      the warp group g = warp / 4 takes product g (NPR = 2; NPR = 1: group 0 alone)
    auto epilogue = [&](int b, const TcWork<NPR> &w, const int (&fixab)[NPR]) {
        const int g = NT == 256 ? warp >> 2 : 0, wq = warp & 3;
        if (NT == 256 && NPR == 1 && g == 1) return;
        const uint32_t lane_addr = tmem + (uint32_t)(b * LA * G::NB) + ((uint32_t)(wq * 32) << 16);
        // accumulator row of this thread (MM = 64: lanes 16..31 of each warp hold nothing)
        const int rrow = MM == 128 ? 32 * wq + lane : 16 * warp + lane;
        const bool rowok = MM == 128 || lane < 16;
        const bool lead = (tid & 127) == 0;                // owns c[0] of its group's product
#pragma unroll
        for (int pp = 0; pp < NPR; pp++) {
            if (NT == 256 && NPR == 2 && pp != g) continue;
            int v[LA][G::PCOL / 16][16];
#pragma unroll
            for (int l = 0; l < LA; l++)
#pragma unroll
                for (int c16 = 0; c16 < G::PCOL / 16; c16++)
                    tmem_ld16(lane_addr + l * G::NB + pp * G::PCOL + 16 * c16, v[l][c16]);
            tmem_ld_wait();
            const long long orow = w.orow[pp];
            auto comb = [&](int t) {     // limb recombination of D column t (exact in int32)
                auto D = [&](int l, int lb) { const int col = lb * G::NL + t; return v[l][col >> 4][col & 15]; };
                if (LA == 1 && LB == 1) return D(0, 0);
                if (LA == 1) return (64 * D(0, 0) + D(0, 1)) % M;
                if (LB == 1) return (64 * D(0, 0) + D(1, 0)) % M;
                return (4096 * (D(0, 0) % M) + 64 * (D(0, 1) + D(1, 0)) + D(1, 1)) % M;
            };
            int fix = 0;                                   // = D(p-1), for the c[0] owner
            const int w0 = 4 * g;                          // first warp of this group
            {
                if constexpr (G::FIXROW) {
                    if (warp == w0) fix = __shfl_sync(FULL, comb(G::NT), G::R0);
                } else {
                    // D(p-1) lives in accumulator row (p-1) mod MM of block (p-1)/MM
                    constexpr int RS = (P - 1) % MM, TS = (P - 1) / MM;
                    constexpr int WS = MM == 128 ? RS / 32 : RS / 16;
                    constexpr int LS = MM == 128 ? RS % 32 : RS % 16;
                    if (warp == w0 + WS && lane == LS) fixs[pp] = comb(TS);
                    if (WS == 0) __syncwarp();
                    else if (warp == w0 || warp == w0 + WS) {
                        if (g == 0) asm volatile("bar.sync 1, 64;" ::: "memory");
                        else asm volatile("bar.sync 2, 64;" ::: "memory");
                    }
                    if (lead) fix = fixs[pp];
                }
            }
            if (orow < 0 || !rowok) continue;
            auto store = [&](auto *op) {
                constexpr int OSTRIDE = sizeof(*op) == 2 ? PS::P8 : PS::P16;
#pragma unroll
                for (int t = 0; t < G::NT; t++) {
                    const int k = MM * t + rrow;
                    if (k >= OSTRIDE) break;
                    int x = comb(t);
                    if (k == 0) x = x - fix + (NT == 256 ? fixab_s[b * NPR + pp] : fixab[pp]) % M;
                    int vv = k < P ? canon<M>(x) : 0;
                    if (XOPS && a.round3) vv -= canon<3>(vv);      // encapsulation's Round
                    op[k] = (std::remove_reference_t<decltype(*op)>)vv;
                }
            };
            uint8_t *orp = (pp == 1 && a.out2) ? (uint8_t *)a.out2 + orow * a.out2_stride * a.out_bytes
                                               : (uint8_t *)a.out + orow * a.out_stride * a.out_bytes;
            if (a.out_bytes == 2) store(reinterpret_cast<int16_t *>(orp));
            else store(reinterpret_cast<int8_t *>(orp));
        }
    };

    // ES (big x big only): the next item is staged (registers -> hA / Z staging, which the MMAs
    // do not read) while this item's MMAs run; its rows were prefetched one iteration earlier.
    // Elsewhere the second item's live state costs registers and CTAs per SM (80 -> 87 for
    // big x small: 6 -> 5).
    constexpr bool ES = LA == 2 && LB == 2;
    if constexpr (ST == 1 && !ES) {
        prefetch(blockIdx.x);
        for (long long it = blockIdx.x; it < a.n_out; it += gridDim.x) {
            const TcWork<NPR> w = wn;
            int fixab[NPR];                               // a[p-1] b[p-1] (thread 0)
            stage(w, fixab, 0);
            __syncthreads();
            build(0);
            tc_fence_before();
            __syncthreads();
            if (warp == 0) issue(0);
            prefetch(it + gridDim.x);
            if (tid == 0) mbar_wait(bar, phases & 1u);
            phases ^= 1u;
            __syncthreads();
            tc_fence_after();
            epilogue(0, w, fixab);
            tc_fence_before();   // TMEM reads ordered before the next item's MMAs (issued after later barriers)
        }
    } else if constexpr (ST == 1) {
        long long it = blockIdx.x;
        if (it < a.n_out) {
            prefetch(it);
            TcWork<NPR> cur = wn;
            int fcur[NPR];                                // a[p-1] b[p-1] (thread 0)
            stage(cur, fcur, 0);
            prefetch(it + gridDim.x);
            for (; it < a.n_out; it += gridDim.x) {
                const long long nx = it + gridDim.x;
#pragma unroll 1
                for (int h = 0; h < NH - 1; h++) {        // all parts but the last: build, MMAs, wait
                    __syncthreads();                      // staging complete / previous part's MMAs done
                    build(0, h);
                    tc_fence_before();
                    __syncthreads();
                    if (warp == 0) issue(0, h);
                    if (tid == 0) mbar_wait(bar, phases & 1u);
                    phases ^= 1u;
                }
                __syncthreads();                          // staging of item it complete
                build(0, NH - 1);
                tc_fence_before();
                __syncthreads();                          // operands built; staging area free
                if (warp == 0) issue(0, NH - 1);
                const TcWork<NPR> nxt = wn;
                int fnx[NPR];
#pragma unroll
                for (int pp = 0; pp < NPR; pp++) fnx[pp] = 0;
                if (nx < a.n_out) {
                    stage(nxt, fnx, 0);
                    prefetch(nx + gridDim.x);
                }
                if (tid == 0) mbar_wait(bar, phases & 1u);
                phases ^= 1u;
                __syncthreads();
                tc_fence_after();
                epilogue(0, cur, fcur);
                tc_fence_before();   // TMEM reads ordered before the next item's MMAs (issued after later barriers)
                cur = nxt;
#pragma unroll
                for (int pp = 0; pp < NPR; pp++) fcur[pp] = fnx[pp];
            }
        }
    } else {
        long long it = blockIdx.x;
        if (it < a.n_out) {
            prefetch(it);
            TcWork<NPR> cur = wn;
            int fcur[NPR];
            stage(cur, fcur, 0);
            __syncthreads();
            build(0);
            tc_fence_before();
            __syncthreads();
            if (warp == 0) issue(0);
            prefetch(it + gridDim.x);
            int b = 0;
            for (; it < a.n_out; it += gridDim.x) {
                const long long nx = it + gridDim.x;
                TcWork<NPR> nxt = wn;
                int fnx[NPR];
#pragma unroll
                for (int pp = 0; pp < NPR; pp++) fnx[pp] = 0;
                if (nx < a.n_out) {
                    // item nx into stage b^1 while item it's MMAs run (stage b^1's previous MMAs
                    // completed one iteration ago; the staging area was last read by build before
                    // the previous barrier)
                    stage(nxt, fnx, b ^ 1);
                    __syncthreads();
                    build(b ^ 1);
                    tc_fence_before();
                    prefetch(nx + gridDim.x);
                }
                if (tid == 0) mbar_wait(bar + b, (phases >> b) & 1u);
                phases ^= 1u << b;
                __syncthreads();                          // also: stage b^1 complete
                tc_fence_after();
                // issue item nx's MMAs before this item's epilogue (thread 0 may block in the
                // issue until the tensor pipe accepts them; the other warps go on)
                if (warp == 0 && nx < a.n_out) issue(b ^ 1);
                epilogue(b, cur, fcur);
                tc_fence_before();
                cur = nxt;
#pragma unroll
                for (int pp = 0; pp < NPR; pp++) fcur[pp] = fnx[pp];
                b ^= 1;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)TCOLS));
}

// shared memory of a tc_mul_kernel instantiation (ST operand stages)
template <class G, int LA, int LB, int NPR, int ST, int MM = 128, int NH = 1>
constexpr int tc_smem_bytes() {
    using H = TcParts<G, LA, LB, NPR, MM, NH>;
    return ST * (LA * H::A_BYTES + H::B_BYTES) + LA * G::HA_LEN + NPR * LB * G::Z_LEN + 128;
}
template <class G, int LA, int ST>
constexpr int tc_tmem_cols() {
    return ST * LA * G::NB <= 32 ? 32 : ST * LA * G::NB <= 64 ? 64 : ST * LA * G::NB <= 128 ? 128 : 256;
}

}  // namespace sntrup
