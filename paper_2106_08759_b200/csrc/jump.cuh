// jump.cuh -- R/q root inversion by jump-divsteps (App. D "jump-div-step"; the
// constant-time extended GCD of [BY19]).
//
// The divstep recipe is the one of divstep.cuh (C15): state (delta, f, g, v, r), p+1
// coefficients, exactly 2p-1 steps, 1/a = f0^-1 * reverse(v).  A jump of s <= 31 steps is taken
// in two parts:
//
//  1. decisions: the s steps only read coefficient 0 of f and g, and coefficient 0 after t steps
//     depends only on coefficients 0..t of the start, so one warp (lane i = coefficient i of a
//     32-coefficient window of f, g) runs the s steps on the window and accumulates the 2x2
//     transition matrix U (entries polynomials of degree <= s, lane j = coefficient j):
//         x^s f' = u00 f + u01 g,      x^s g' = u10 f + u11 g,
//     per step: rows swapped on a swap, row1 <- f0 row1 - g0 row0, row0 <- x row0.
//     The (v, r) pair moves by the conjugate W = diag(1, x) U diag(1, 1/x) (both recurrences are
//     left products of per-step matrices S', S with S' diag(1,x) = diag(1,x) S):
//         v' = u00 v + (u01 / x) r,    r' = (x u10) v + u11 r     (u01 is divisible by x).
//  2. application of U to the whole of f, g, v, r: 4 * 32 multiply-adds per output coefficient
//     pair, exact int32 sums (64 |u| |c| <= 64 * 3940^2 < 2^30), R = 2 outputs per thread.
//
// Layout: one 2-CTA cluster per root.  CTA 0: warp 0 decides; warps on SMSPs 1-3 apply U to f, g
// (SMSP 0 is left to the decision warp: its chain is latency bound and must not queue behind the
// appliers' IMADs).  CTA 1 applies U to v, r: (v, r) never feed back into the decisions, so it is
// a pure consumer of the U's, which CTA 0 stores into its shared memory (DSMEM, one slot per
// jump) and signals with a per-jump mbarrier.  The decision warp runs one jump ahead: while f, g
// get jump k, it computes the low 32 coefficients of the next f, g itself (from coefficients
// 0..62 of the current ones and U_k) and runs the decisions of jump k+1; named barriers hand U_k
// to CTA 0's appliers (bar 1) and report their application complete (bar 2).
//
// One step's chain: D = f0 g - g0 f is computed before the swap decision is known (a swap only
// flips its sign: with (f, g, f0, g0) exchanged, f0 g - g0 f becomes -D), likewise row1's update.
//
// Constant time: every trip count and address depends on p and the jump index only.  Known-zero
// work is skipped with data-independent bounds: after n steps len(f), len(g) <= min(p+1, 2p+1-n)
// (their sum drops by one per step, [BY19] Thm 6.2 for polynomials) and len(v), len(r) <=
// min(p+1, n+1) (clipped at p+1 as in C15; clipping commutes with the x-power products since
// none moves a coefficient to a lower index).
#pragma once
#include "common.cuh"
#include "divstep.cuh"

#ifndef SNTRUP_JUMP_RF
#define SNTRUP_JUMP_RF 2          // (f, g) outputs per applier item (2 or 4; A/B)
#endif
#ifndef SNTRUP_JUMP_PREP4
#define SNTRUP_JUMP_PREP4 1       // prep sums in 4 independent chains (3.1k vs 3.2k cycles per jump)
#endif
#ifndef SNTRUP_JUMP_CHUNKED
#define SNTRUP_JUMP_CHUNKED 0     // appliers' tap loop rolled in chunks of 8 (A/B: not faster)
#endif
#ifndef SNTRUP_JUMP_UNROLL
#define SNTRUP_JUMP_UNROLL 8      // decision-loop unroll factor: 4-8 (3.1-3.2k cycles per jump) beats
                                  // full unrolling (4.0k: the 16 KB loop thrashes the instruction
                                  // caches shared with the appliers) and 1 (3.6k)
#endif
#ifndef SNTRUP_JUMP_MODE
#define SNTRUP_JUMP_MODE 0        // timing experiments: 1 = decisions only, 2 = applications only
#endif

#ifndef SNTRUP_JUMP_TRACE
#define SNTRUP_JUMP_TRACE 0       // 1: the decision warp of root 0 records clock64 per jump phase
#endif

namespace sntrup {

#if SNTRUP_JUMP_TRACE
__device__ long long g_jump_trace[128][8];
#define JTRACE(k, i)                                                          \
    do {                                                                      \
        if (blockIdx.x == 0 && lane == 0 && (k) < 128) g_jump_trace[k][i] = clock64(); \
    } while (0)
#else
#define JTRACE(k, i) do { } while (0)
#endif

__device__ __forceinline__ void named_bar_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cta address -> the same offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_rank(const void *p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"((uint32_t)__cvta_generic_to_shared(p)), "r"(rank));
    return r;
}
// asynchronous store into another CTA's shared memory, completing `bytes` of the transaction
// count of that CTA's mbarrier (the issuing thread does not wait)
__device__ __forceinline__ void st_async_v4(uint32_t ra, int4 v, uint32_t ra_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.s32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(ra),
                 "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(ra_bar)
                 : "memory");
}
__device__ __forceinline__ void st_async_v2(uint32_t ra, int x, int y, uint32_t ra_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.s32 [%0], {%1, %2}, [%3];" ::"r"(ra), "r"(x),
                 "r"(y), "r"(ra_bar)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t phase) {
    const long long t0 = clock64();
    for (;;) {
        uint32_t ok;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}\n"
            : "=r"(ok)
            : "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(phase)
            : "memory");
        if (ok) return;
        if (clock64() - t0 > (1LL << 31)) __trap();
    }
}

// |x| < 2^30 -> centered representative in [-(M-1)/2, (M-1)/2] (float quotient estimate, off
// by at most one, then one correction)
template <int M>
__device__ __forceinline__ int ired(int x) {
    const int k = __float2int_rn(__int2float_rn(x) * (1.0f / (float)M));
    int r = x - k * M;
    r += (r < -(M - 1) / 2) ? M : 0;
    r -= (r > (M - 1) / 2) ? M : 0;
    return r;
}

template <class PS, int M>
struct RqJump {
    static constexpr int P = PS::P, P1 = P + 1, S = 2 * P - 1;
    static constexpr int J = 31;                               // steps per jump (U: 32 coefficients)
    static constexpr int UNR = SNTRUP_JUMP_UNROLL;
    static constexpr bool CHUNKED = SNTRUP_JUMP_CHUNKED;     // appliers' tap loop rolled in chunks of 8
    static constexpr int NJ = (S + J - 1) / J;
    static constexpr int NT = 512;
    static constexpr int NA0 = 384;                            // CTA 0 appliers: warps on SMSPs 1-3
    static constexpr int NB0 = 32 + NA0;                       // CTA 0 named-barrier count
    static constexpr int NA1 = NT;                             // CTA 1: every warp applies
    static constexpr int R = 2;                                // outputs per applier item
    static constexpr int PAD = 32;                             // zeros below index 0
    static constexpr int P1R = (P1 + 3) / 4 * 4;
    static constexpr int LEN = PAD + P1R + 36;                 // f, g windows reach P1R + 32
    static constexpr bool ONE_RED = 2LL * ((M + 1) / 2) * ((M + 1) / 2) < (1LL << 24);
    // dynamic shared memory (both CTAs use the same layout, each a part of it)
    static constexpr int OFF_BUF = 0;                          // int [2][2][LEN]: CTA 0 f, g / CTA 1 v, r
    static constexpr int OFF_U = OFF_BUF + 2 * 2 * LEN * 4;    // int4 [NJ][32]: CTA 0 uses slots 0, 1
    static constexpr int OFF_BAR = OFF_U + NJ * 32 * 16;       // uint64 [NJ] (CTA 1)
    static constexpr int OFF_FIN = OFF_BAR + NJ * 8;           // int [2]: f0, delta (CTA 1, with U_{NJ-1})
    static constexpr int SMEM_USED = OFF_FIN + 16;
    // reserved per CTA: more than half an SM's shared memory, so each CTA of the pair has its SM
    // to itself (the decision chain must not share issue slots with another kernel's CTAs)
    static constexpr int SMEM = SMEM_USED > 116 * 1024 ? SMEM_USED : 116 * 1024;
    static_assert(LEN % 4 == 0 && PAD % 4 == 0, "16-byte aligned rows");
    static_assert(R == 2, "items of two outputs (8-byte window loads)");

    // a x - b y (mod M), float-held exact integers (as Divstep)
    __device__ __forceinline__ static float mulsub(float a, float x, float b, float y) {
        if (ONE_RED) return fmodc<M>(__fmaf_rn(a, x, -__fmul_rn(b, y)));
        return fmodc<M>(__fmaf_rn(-b, y, fmodc<M>(__fmul_rn(a, x))));
    }

    static __host__ __device__ constexpr int steps(int k) { return S - J * k < J ? S - J * k : J; }
    static __host__ __device__ constexpr int rup4(int x) { return (x + 3) / 4 * 4; }
    // f, g length bound before jump k (outputs computed), v, r length bound after it
    static __host__ __device__ constexpr int fg_len(int k) {
        return k < 0 ? P1R : rup4((2 * P + 1 - J * k) < P1 ? (2 * P + 1 - J * k) : P1);
    }
    static __host__ __device__ constexpr int vr_len(int k) {
        return rup4((J * k + steps(k) + 1) < P1 ? (J * k + steps(k) + 1) : P1);
    }

    // s divsteps on the window (lane = coefficient); U_k -> u[4] (float-held ints); f0 is the
    // uniform f_0 (updated), delta the uniform delta
    template <int SC>
    __device__ __forceinline__ static void decide(float Ff, float Gf, float &f0, int &delta, int s, int lane,
                                                  float (&u)[4]) {
        float u00 = lane == 0 ? 1.0f : 0.0f, u01 = 0.0f, u10 = 0.0f, u11 = u00;
        float g0 = __shfl_sync(FULL, Gf, 0);
#pragma unroll (UNR)
        for (int t = 0; t < (SC ? SC : J); t++) {
            if (!SC && t >= s) break;
            const float D = mulsub(f0, Gf, g0, Ff);                     // f0 g - g0 f (pre-swap)
            const float E0 = mulsub(f0, u10, g0, u00);                  // f0 row1 - g0 row0
            const float E1 = mulsub(f0, u11, g0, u01);
            const bool sw = (delta > 0) && (g0 != 0.0f);
            const float T = sw ? -D : D;                                // the new g (before / x)
            const float gn = __shfl_sync(FULL, T, 1);                   // next g_0
            const float Gn = __shfl_down_sync(FULL, T, 1);              // g <- g / x
            const float a0 = sw ? u10 : u00, a1 = sw ? u11 : u01;       // row0 after the swap
            const float x0 = __shfl_up_sync(FULL, a0, 1), x1 = __shfl_up_sync(FULL, a1, 1);
            Ff = sw ? Gf : Ff;
            f0 = sw ? g0 : f0;
            delta = sw ? 1 - delta : delta + 1;
            u10 = sw ? -E0 : E0;
            u11 = sw ? -E1 : E1;
            u00 = lane ? x0 : 0.0f;                                     // row0 <- x row0
            u01 = lane ? x1 : 0.0f;
            Gf = Gn;
            g0 = gn;
        }
        u[0] = u00; u[1] = u01; u[2] = u10; u[3] = u11;
    }

    // f, g application of jump k (CTA 0): outputs n .. n+RR-1 (RR = 2: 8-byte window loads, 4:
    // 16-byte loads)
    template <bool FULLJ, int RR>
    __device__ __forceinline__ static void apply_fg(const int *Fb, const int *Gb, int *Fo, int *Go,
                                                    const int4 *U, int n, int s) {
        constexpr int WN = RR + 32;                                 // window F[n+s-31 .. n+s+RR]
        if constexpr (FULLJ && RR == 2 && CHUNKED) {
            // taps in rolled chunks of 8 (small code: the decision warp's loop and this one stay
            // in the instruction caches); window of chunk c: F[n + 24 - 8c .. n + 33 - 8c]
            int aF0 = 0, aF1 = 0, aG0 = 0, aG1 = 0;
#pragma unroll 1
            for (int c = 0; c < 4; c++) {
                int wF[10], wG[10];
#pragma unroll
                for (int w = 0; w < 10; w += 2) {
                    const int2 x = *reinterpret_cast<const int2 *>(Fb + n + 24 - 8 * c + w);
                    const int2 y = *reinterpret_cast<const int2 *>(Gb + n + 24 - 8 * c + w);
                    wF[w] = x.x; wF[w + 1] = x.y; wG[w] = y.x; wG[w + 1] = y.y;
                }
#pragma unroll
                for (int jj = 0; jj < 8; jj++) {
                    const int4 w = U[8 * c + jj];
                    aF0 += w.x * wF[7 - jj] + w.y * wG[7 - jj];
                    aG0 += w.z * wF[7 - jj] + w.w * wG[7 - jj];
                    aF1 += w.x * wF[8 - jj] + w.y * wG[8 - jj];
                    aG1 += w.z * wF[8 - jj] + w.w * wG[8 - jj];
                }
            }
            *reinterpret_cast<int2 *>(Fo + n) = make_int2(ired<M>(aF0), ired<M>(aF1));
            *reinterpret_cast<int2 *>(Go + n) = make_int2(ired<M>(aG0), ired<M>(aG1));
            return;
        }
        int wF[WN], wG[WN];
        if (FULLJ) {                                                // s = 31: window starts at n
            if constexpr (RR == 4) {
#pragma unroll
                for (int w = 0; w < WN; w += 4) {
                    const int4 x = *reinterpret_cast<const int4 *>(Fb + n + w);
                    const int4 y = *reinterpret_cast<const int4 *>(Gb + n + w);
                    wF[w] = x.x; wF[w + 1] = x.y; wF[w + 2] = x.z; wF[w + 3] = x.w;
                    wG[w] = y.x; wG[w + 1] = y.y; wG[w + 2] = y.z; wG[w + 3] = y.w;
                }
            } else {
#pragma unroll
                for (int w = 0; w < WN; w += 2) {
                    const int2 x = *reinterpret_cast<const int2 *>(Fb + n + w);
                    const int2 y = *reinterpret_cast<const int2 *>(Gb + n + w);
                    wF[w] = x.x; wF[w + 1] = x.y; wG[w] = y.x; wG[w + 1] = y.y;
                }
            }
        } else {
#pragma unroll
            for (int w = 0; w < WN; w++) { wF[w] = Fb[n + s - 31 + w]; wG[w] = Gb[n + s - 31 + w]; }
        }
        int aF[RR], aG[RR];
#pragma unroll
        for (int m = 0; m < RR; m++) { aF[m] = 0; aG[m] = 0; }
#pragma unroll
        for (int j = 0; j < 32; j++) {
            const int4 w = U[j];
#pragma unroll
            for (int m = 0; m < RR; m++) {
                const int fv = wF[m + 31 - j], gv = wG[m + 31 - j];
                aF[m] += w.x * fv + w.y * gv;
                aG[m] += w.z * fv + w.w * gv;
            }
        }
        if constexpr (RR == 4) {
            *reinterpret_cast<int4 *>(Fo + n) = make_int4(ired<M>(aF[0]), ired<M>(aF[1]), ired<M>(aF[2]), ired<M>(aF[3]));
            *reinterpret_cast<int4 *>(Go + n) = make_int4(ired<M>(aG[0]), ired<M>(aG[1]), ired<M>(aG[2]), ired<M>(aG[3]));
        } else {
            *reinterpret_cast<int2 *>(Fo + n) = make_int2(ired<M>(aF[0]), ired<M>(aF[1]));
            *reinterpret_cast<int2 *>(Go + n) = make_int2(ired<M>(aG[0]), ired<M>(aG[1]));
        }
    }

    // v, r application (CTA 1): v'[n+m] = sum u00[j] v[n+m-j] + u01[j] r[n+m+1-j],
    // r'[n+m] = sum u10[j] v[n+m-1-j] + u11[j] r[n+m-j]; windows from n - 32
    __device__ __forceinline__ static void apply_vr(const int *Vb, const int *Rb, int *Vo, int *Ro,
                                                    const int4 *U, int n) {
        if constexpr (CHUNKED) {
            // taps in rolled chunks of 8; chunk c: V[n - 8c - 8 .. n - 8c + 1], R[.. n - 8c + 3]
            int aV0 = 0, aV1 = 0, aR0 = 0, aR1 = 0;
#pragma unroll 1
            for (int c = 0; c < 4; c++) {
                int wV[10], wR[12];
#pragma unroll
                for (int w = 0; w < 12; w += 2) {
                    const int2 y = *reinterpret_cast<const int2 *>(Rb + n - 8 * c - 8 + w);
                    wR[w] = y.x; wR[w + 1] = y.y;
                    if (w < 10) {
                        const int2 x = *reinterpret_cast<const int2 *>(Vb + n - 8 * c - 8 + w);
                        wV[w] = x.x; wV[w + 1] = x.y;
                    }
                }
#pragma unroll
                for (int jj = 0; jj < 8; jj++) {
                    const int4 w = U[8 * c + jj];
                    aV0 += w.x * wV[8 - jj] + w.y * wR[9 - jj];
                    aR0 += w.z * wV[7 - jj] + w.w * wR[8 - jj];
                    aV1 += w.x * wV[9 - jj] + w.y * wR[10 - jj];
                    aR1 += w.z * wV[8 - jj] + w.w * wR[9 - jj];
                }
            }
            if (n + 1 < P1) {
                *reinterpret_cast<int2 *>(Vo + n) = make_int2(ired<M>(aV0), ired<M>(aV1));
                *reinterpret_cast<int2 *>(Ro + n) = make_int2(ired<M>(aR0), ired<M>(aR1));
            } else if (n < P1) {
                Vo[n] = ired<M>(aV0);
                Ro[n] = ired<M>(aR0);
            }
            return;
        }
        constexpr int WV = R + 32, WR = R + 34;
        int wV[WV], wR[WR];
#pragma unroll
        for (int w = 0; w < WR; w += 2) {
            const int2 y = *reinterpret_cast<const int2 *>(Rb + n - 32 + w);
            wR[w] = y.x; wR[w + 1] = y.y;
            if (w < WV) {
                const int2 x = *reinterpret_cast<const int2 *>(Vb + n - 32 + w);
                wV[w] = x.x; wV[w + 1] = x.y;
            }
        }
        int aV[R], aR[R];
#pragma unroll
        for (int m = 0; m < R; m++) { aV[m] = 0; aR[m] = 0; }
#pragma unroll
        for (int j = 0; j < 32; j++) {
            const int4 w = U[j];
#pragma unroll
            for (int m = 0; m < R; m++) {
                aV[m] += w.x * wV[m + 32 - j] + w.y * wR[m + 33 - j];
                aR[m] += w.z * wV[m + 31 - j] + w.w * wR[m + 32 - j];
            }
        }
        // clipped at index p (C15): outputs beyond stay zero
        if (n + 1 < P1) {
            *reinterpret_cast<int2 *>(Vo + n) = make_int2(ired<M>(aV[0]), ired<M>(aV[1]));
            *reinterpret_cast<int2 *>(Ro + n) = make_int2(ired<M>(aR[0]), ired<M>(aR[1]));
        } else if (n < P1) {
            Vo[n] = ired<M>(aV[0]);
            Ro[n] = ired<M>(aR[0]);
        }
    }
};

// One root per 2-CTA cluster: row `row` of a.in -> a.out, a.ok.
template <class PS, int M>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(RqJump<PS, M>::NT, 1) jump_cluster_kernel(InvArgs a) {
    using JS = RqJump<PS, M>;
    constexpr int P = PS::P, NT = JS::NT, PAD = JS::PAD, LEN = JS::LEN, NJ = JS::NJ, R = JS::R;
    constexpr int RF = SNTRUP_JUMP_RF;
    extern __shared__ __align__(16) uint8_t smem[];
    int *buf = reinterpret_cast<int *>(smem + JS::OFF_BUF);           // [parity][poly][LEN]
    int4 *Us = reinterpret_cast<int4 *>(smem + JS::OFF_U);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + JS::OFF_BAR);
    int *fin = reinterpret_cast<int *>(smem + JS::OFF_FIN);
    auto B = [&](int par, int poly) { return buf + (par * 2 + poly) * LEN + PAD; };
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = cluster_rank();
    const long long row = (long long)(blockIdx.x >> 1);

    for (int i = tid; i < 2 * 2 * LEN; i += NT) buf[i] = 0;
    __syncthreads();
    if (rank == 0) {
        for (int i = tid; i <= P; i += NT) {
            B(0, 0)[i] = (i == 0) ? 1 : ((i == P - 1 || i == P) ? -1 : 0);   // f = 1 - x^(p-1) - x^p
            B(0, 1)[i] = (i < P) ? load_coef(a.in, row, P - 1 - i) : 0;     // g_i = a_(p-1-i)
        }
    } else {
        if (tid == 0) B(0, 1)[0] = 1;                                       // r = 1 (v = 0)
        // barrier k: one arrival (armed here) + the 512 bytes of U_k (+ 8 bytes f0, delta for the last)
        if (tid < NJ) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bars + tid)),
                         "r"(1) : "memory");
            mbar_arrive_expect_tx(bars + tid, 32 * 16 + (tid == NJ - 1 ? 8 : 0));
        }
        if (tid == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    cluster_sync_all();                                                    // CTA 1's barriers visible

    if (rank == 0) {
        if (warp == 0) {
            // ---------------------------------------------------------------- decision warp
            float Ff = (float)B(0, 0)[lane], Gf = (float)B(0, 1)[lane], f0 = 1.0f;
            int delta = 1;
#pragma unroll 1
            for (int k = 0; k < NJ; k++) {
                const int s = JS::steps(k), b = k & 1;
                float u[4];
                JTRACE(k, 0);
#if SNTRUP_JUMP_MODE == 2
                u[0] = lane == 0; u[1] = 0; u[2] = 0; u[3] = lane == 0; (void)Gf;
#else
                if (s == JS::J) JS::template decide<JS::J>(Ff, Gf, f0, delta, s, lane, u);
                else JS::template decide<0>(Ff, Gf, f0, delta, s, lane, u);
#endif
                const int4 uk = make_int4((int)u[0], (int)u[1], (int)u[2], (int)u[3]);
                JTRACE(k, 1);
                // to CTA 1 (slot k) and its barrier k; the last one carries f0 and delta
                const uint32_t rbar = map_rank(bars + k, 1);
                if (k + 1 == NJ && lane == 0) st_async_v2(map_rank(fin, 1), (int)f0, delta, rbar);
                st_async_v4(map_rank(Us + k * 32 + lane, 1), uk, rbar);
                JTRACE(k, 4);
                if (k > 0) named_bar_sync(2, JS::NB0);                     // f, g of jump k-1 applied
                JTRACE(k, 2);
                Us[b * 32 + lane] = uk;
                __syncwarp();
                named_bar_arrive(1, JS::NB0);                              // U_k to CTA 0's appliers
                if (k + 1 < NJ) {
                    // low 32 coefficients of the next f, g: f'[i] = sum_j u00[j] f[i+s-j] + u01[j] g[i+s-j]
                    const int *Fb = B(b, 0) + lane + s, *Gb = B(b, 1) + lane + s;
#if SNTRUP_JUMP_PREP4
                    int af[4] = {0, 0, 0, 0}, ag[4] = {0, 0, 0, 0};             // 4 chains each
#pragma unroll
                    for (int j = 0; j < 32; j++) {
                        const int4 w = Us[b * 32 + j];
                        const int fv = Fb[-j], gv = Gb[-j];
                        af[j & 3] += w.x * fv + w.y * gv;
                        ag[j & 3] += w.z * fv + w.w * gv;
                    }
                    Ff = (float)ired<M>((af[0] + af[1]) + (af[2] + af[3]));
                    Gf = (float)ired<M>((ag[0] + ag[1]) + (ag[2] + ag[3]));
#else
                    int af = 0, ag = 0;
#pragma unroll
                    for (int j = 0; j < 32; j++) {
                        const int4 w = Us[b * 32 + j];
                        const int fv = Fb[-j], gv = Gb[-j];
                        af += w.x * fv + w.y * gv;
                        ag += w.z * fv + w.w * gv;
                    }
                    Ff = (float)ired<M>(af);
                    Gf = (float)ired<M>(ag);
#endif
                }
                JTRACE(k, 3);
            }
        } else if ((warp & 3) != 0) {
            // ---------------------------------------------------------------- f, g appliers
            const int ta = 32 * (warp - 1 - (warp >> 2)) + lane;
#pragma unroll 1
            for (int k = 0; k < NJ; k++) {
                named_bar_sync(1, JS::NB0);                                // U_k
                if (warp == 1) JTRACE(k, 5);
                const int s = JS::steps(k), b = k & 1, o = b ^ 1;
                const int A = JS::fg_len(k), Aold = JS::fg_len(k - 2);
                const int4 *U = Us + b * 32;
#if SNTRUP_JUMP_MODE == 1
                const int nit = 0;
#else
                const int nit = A / RF;
#endif
#pragma unroll 1
                for (int it = ta; it < nit; it += JS::NA0) {
                    if (s == JS::J) JS::template apply_fg<true, RF>(B(b, 0), B(b, 1), B(o, 0), B(o, 1), U, RF * it, s);
                    else JS::template apply_fg<false, RF>(B(b, 0), B(b, 1), B(o, 0), B(o, 1), U, RF * it, s);
                }
                // beyond this jump's bound: clear what jump k-2 left in this buffer
                for (int i = A + ta; i < Aold; i += JS::NA0) {
                    B(o, 0)[i] = 0;
                    B(o, 1)[i] = 0;
                }
                if (warp == 1) JTRACE(k, 6);
                if (k + 1 < NJ) named_bar_arrive(2, JS::NB0);             // jump k applied
            }
        }
    } else {
        // -------------------------------------------------------------------- v, r appliers
#pragma unroll 1
        for (int k = 0; k < NJ; k++) {
            mbar_wait_cluster(bars + k, 0);
            const int b = k & 1, o = b ^ 1;
#if SNTRUP_JUMP_MODE == 1
            const int nit = 0;
#else
            const int nit = JS::vr_len(k) / R;
#endif
#pragma unroll 1
            for (int it = tid; it < nit; it += JS::NA1)
                JS::apply_vr(B(b, 0), B(b, 1), B(o, 0), B(o, 1), Us + k * 32, R * it);
            __syncthreads();
        }
        // 1/a = f0^-1 reverse(v)
        const int f0 = fin[0], delta = fin[1];
        const bool ok = delta == 0;
        const int fr = ((f0 % M) + M) % M;
        const int sc = inv_mod_const<M>(fr == 0 ? 1 : fr);
        const int *V = B(NJ & 1, 0);
        const int ostride = a.out_bytes == 2 ? PS::P8 : PS::P16;
        for (int k = tid; k < ostride; k += NT) {
            int val = 0;
            if (k < P && ok) val = canon<M>(sc * V[P - 1 - k]);
            if (a.out_bytes == 2) ((int16_t *)a.out)[row * a.out_stride + k] = (int16_t)val;
            else ((int8_t *)a.out)[row * a.out_stride + k] = (int8_t)val;
        }
        if (tid == 0 && a.ok) a.ok[row] = ok ? 1 : 0;
    }
    cluster_sync_all();       // no CTA leaves while the other may still touch its shared memory
}

template <class PS, int M>
cudaError_t launch_jump_roots(const InvArgs &a, cudaStream_t s, bool reserve_sm = true) {
    using JS = RqJump<PS, M>;
    static unsigned long long attr_set = 0;         // per device (bit)
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr_set >> (dev & 63) & 1ull)) {
        cudaError_t e = cudaFuncSetAttribute(jump_cluster_kernel<PS, M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             JS::SMEM);
        if (e != cudaSuccess) return e;
        attr_set |= 1ull << (dev & 63);
    }
    jump_cluster_kernel<PS, M><<<(unsigned)(2 * a.n), JS::NT, reserve_sm ? JS::SMEM : JS::SMEM_USED, s>>>(a);
    return cudaGetLastError();
}

}  // namespace sntrup
