// divstep.cuh -- constant-time inversion in (Z/M)[x]/(x^p - x - 1), M = 3 or q, one warp per
// element.
//
// The paper's single inversions (the root of each batchInv tree; R/q inversion
// cost P:7063-7080) use the constant-time extended GCD of Bernstein-Yang [BY19] cited at
// P:3562-3567.  This is the divstep recipe of DESIGN.md C15: state (delta, f, g, v, r) with
// p+1 coefficients, exactly 2p-1 iterations, branch-free in the data (the swap is a
// warp-uniform select on public-size registers).  The element is invertible iff delta == 0
// at the end; then 1/a = f0^{-1} * reverse(v).
//
// Layout: lane l holds coefficients l*C .. l*C+C-1 of each vector (C = ceil((p+1)/32)) as
// floats holding exact integers; products/reductions are exact single-rounding FMAs
// (|values| <= (M+1)/2, |f0*g - g0*f| < 2^24, see fmodc).
#pragma once
#include "common.cuh"
#include "sample.cuh"

namespace sntrup {

template <class PS, int M>
struct Divstep {
    static constexpr int P = PS::P;
    static constexpr int C = (P + 1 + 31) / 32;
    // single reduction is exact iff 2*((M+1)/2)^2 < 2^24
    static constexpr bool ONE_RED = 2LL * ((M + 1) / 2) * ((M + 1) / 2) < (1LL << 24);

    // a[] = lane's reversed-input chunk: g_i = a_{p-1-i}.  On return out[c] holds
    // coefficient (p-1-(l*C+c)) of 1/a (for l*C+c < p) and the function returns delta == 0.
    __device__ __forceinline__ static bool invert(float (&g)[C], float (&out)[C], int lane) {
        float f[C], v[C], r[C];
#pragma unroll
        for (int c = 0; c < C; c++) {
            const int i = lane * C + c;
            f[c] = (i == 0) ? 1.0f : ((i == P - 1 || i == P) ? -1.0f : 0.0f);
            v[c] = 0.0f;
            r[c] = (i == 0) ? 1.0f : 0.0f;
        }
        int delta = 1;
        for (int loop = 0; loop < 2 * P - 1; loop++) {
            // v <- x * v
            const float vtop = __shfl_up_sync(FULL, v[C - 1], 1);
#pragma unroll
            for (int c = C - 1; c > 0; c--) v[c] = v[c - 1];
            v[0] = lane ? vtop : 0.0f;
            float f0 = __shfl_sync(FULL, f[0], 0);
            float g0 = __shfl_sync(FULL, g[0], 0);
            const bool swap = (delta > 0) && (g0 != 0.0f);
            delta = swap ? -delta : delta;
#pragma unroll
            for (int c = 0; c < C; c++) {
                const float tf = f[c], tv = v[c];
                f[c] = swap ? g[c] : tf;
                g[c] = swap ? tf : g[c];
                v[c] = swap ? r[c] : tv;
                r[c] = swap ? tv : r[c];
            }
            {
                const float t = f0;
                f0 = swap ? g0 : f0;
                g0 = swap ? t : g0;
            }
            delta += 1;
#pragma unroll
            for (int c = 0; c < C; c++) {
                if (ONE_RED) {
                    g[c] = fmodc<M>(__fmaf_rn(f0, g[c], -__fmul_rn(g0, f[c])));
                    r[c] = fmodc<M>(__fmaf_rn(f0, r[c], -__fmul_rn(g0, v[c])));
                } else {
                    g[c] = fmodc<M>(__fmaf_rn(-g0, f[c], fmodc<M>(__fmul_rn(f0, g[c]))));
                    r[c] = fmodc<M>(__fmaf_rn(-g0, v[c], fmodc<M>(__fmul_rn(f0, r[c]))));
                }
            }
            // g <- g / x
            const float gnext = __shfl_down_sync(FULL, g[0], 1);
#pragma unroll
            for (int c = 0; c < C - 1; c++) g[c] = g[c + 1];
            g[C - 1] = (lane < 31) ? gnext : 0.0f;
        }
        const float f0 = __shfl_sync(FULL, f[0], 0);
        int f0i = (int)f0 % M;
        if (f0i < 0) f0i += M;
        long long s = 1, b = f0i, e = M - 2;                // Fermat: f0^(M-2)
        while (e) { if (e & 1) s = s * b % M; b = b * b % M; e >>= 1; }
#pragma unroll
        for (int c = 0; c < C; c++) out[c] = (float)canon<M>((int)s * (int)v[c]);
        return delta == 0;
    }
};

// ---------------------------------------------------------------------------------------------
// R/3 divsteps, bitsliced: the same C15 recipe with every vector held as GF(3) bit planes
// (pl, mi), 32 coefficients per word, word w on lane w % 32 (slot w / 32).  A step is ~45 LOP3 /
// SEL / SHF ops per word plus 3 shuffles, instead of ~16 float ops per coefficient.  Capacity
// 32*W coefficients (W = ceil((p+1)/32)), the same as the float version; bits shifted past it
// are dropped.  f0 is always +-1 (its own inverse in Z/3).
// ---------------------------------------------------------------------------------------------
// Root inversion kernel: one warp per row of `in`; writes `out` rows (int8 or int16) and
// ok[row] = 1 / 0.  Non-invertible rows get zero output.
struct InvArgs {
    long long n;
    RowDesc in;
    void *out;
    long long out_stride;
    int out_bytes;
    uint8_t *ok;
};

template <class PS>
struct R3Divstep {
    static constexpr int P = PS::P;
    static constexpr int W = (P + 1 + 31) / 32;
    static constexpr int NWL = (W + 31) / 32;

    // v <- x v across words (lane l, slot h holds word 32h + l)
    __device__ __forceinline__ static void shift_up(uint32_t (&x)[NWL], int lane) {
        const int src = (lane + 31) & 31;
        uint32_t c[NWL];
#pragma unroll
        for (int h = 0; h < NWL; h++) c[h] = __shfl_sync(FULL, x[h], src);
#pragma unroll
        for (int h = NWL - 1; h >= 0; h--) {
            const uint32_t carry = lane ? c[h] : (h ? c[h - 1] : 0u);
            x[h] = (x[h] << 1) | (carry >> 31);
        }
    }
    // g <- g / x across words
    __device__ __forceinline__ static void shift_down(uint32_t (&x)[NWL], int lane) {
        const int src = (lane + 1) & 31;
        uint32_t c[NWL];
#pragma unroll
        for (int h = 0; h < NWL; h++) c[h] = __shfl_sync(FULL, x[h], src);
#pragma unroll
        for (int h = 0; h < NWL; h++) {
            const uint32_t carry = lane != 31 ? c[h] : (h + 1 < NWL ? c[h + 1] : 0u);
            x[h] = (x[h] >> 1) | (carry << 31);
        }
    }
    __device__ __forceinline__ static void clip(uint32_t (&x)[NWL], int lane) {
#pragma unroll
        for (int h = 0; h < NWL; h++)
            if (32 * h + lane >= W) x[h] = 0;
    }

    // in: int8 row a (coefficients 0..p-1, centered); out: int8 row (p entries written, pad not
    // touched) = 1/a if invertible.  Returns true iff a is invertible (final delta == 0).
    __device__ static bool invert(const int8_t *__restrict__ in, int8_t *__restrict__ out, int lane) {
        uint32_t fp[NWL], fm[NWL], gp[NWL], gm[NWL], vp[NWL], vm[NWL], rp[NWL], rm[NWL];
#pragma unroll
        for (int h = 0; h < NWL; h++) {
            const int w = 32 * h + lane;
            uint32_t pl = 0, mi = 0;
            if (w < W) {
#pragma unroll 8
                for (int b = 0; b < 32; b++) {
                    const int i = 32 * w + b;                       // g_i = a_{p-1-i}
                    if (i < P) {
                        const int v = in[P - 1 - i];
                        pl |= (uint32_t)(v == 1) << b;
                        mi |= (uint32_t)(v == -1) << b;
                    }
                }
            }
            gp[h] = pl; gm[h] = mi;
            // f = 1 - x^{p-1} - x^p
            uint32_t f_p = 0, f_m = 0;
            if (w == 0) f_p |= 1u;
            if (w == (P - 1) / 32) f_m |= 1u << ((P - 1) & 31);
            if (w == P / 32) f_m |= 1u << (P & 31);
            fp[h] = f_p; fm[h] = f_m;
            vp[h] = 0; vm[h] = 0;
            rp[h] = (w == 0) ? 1u : 0u; rm[h] = 0;
        }
        int delta = 1;
#pragma unroll 1
        for (int it = 0; it < 2 * P - 1; it++) {
            shift_up(vp, lane);
            shift_up(vm, lane);
            clip(vp, lane);
            clip(vm, lane);
            const uint32_t bits = __shfl_sync(FULL, (gp[0] & 1u) | ((gm[0] & 1u) << 1) | ((fp[0] & 1u) << 2) |
                                                        ((fm[0] & 1u) << 3), 0);
            const bool swap = (delta > 0) && (bits & 3u);
            delta = swap ? -delta : delta;
            delta += 1;
            const uint32_t sm = swap ? ~0u : 0u;
#pragma unroll
            for (int h = 0; h < NWL; h++) {
                uint32_t t;
                t = (fp[h] ^ gp[h]) & sm; fp[h] ^= t; gp[h] ^= t;
                t = (fm[h] ^ gm[h]) & sm; fm[h] ^= t; gm[h] ^= t;
                t = (vp[h] ^ rp[h]) & sm; vp[h] ^= t; rp[h] ^= t;
                t = (vm[h] ^ rm[h]) & sm; vm[h] ^= t; rm[h] ^= t;
            }
            // trits f0, g0 after the swap
            const uint32_t g0b = swap ? (bits >> 2) : bits, f0b = swap ? bits : (bits >> 2);
            const bool f0neg = (f0b & 2u) != 0;
            const uint32_t mpos = (g0b & 1u) ? ~0u : 0u, mneg = (g0b & 2u) ? ~0u : 0u;
#pragma unroll
            for (int h = 0; h < NWL; h++) {
                // g <- f0 g - g0 f ; r <- f0 r - g0 v
                uint32_t ap = f0neg ? gm[h] : gp[h], am = f0neg ? gp[h] : gm[h];
                uint32_t bp = (fm[h] & mpos) | (fp[h] & mneg), bm = (fp[h] & mpos) | (fm[h] & mneg);
                gf3_add(ap, am, bp, bm);
                gp[h] = ap; gm[h] = am;
                ap = f0neg ? rm[h] : rp[h]; am = f0neg ? rp[h] : rm[h];
                bp = (vm[h] & mpos) | (vp[h] & mneg); bm = (vp[h] & mpos) | (vm[h] & mneg);
                gf3_add(ap, am, bp, bm);
                rp[h] = ap; rm[h] = am;
            }
            shift_down(gp, lane);
            shift_down(gm, lane);
        }
        const bool f0neg = (__shfl_sync(FULL, fm[0] & 1u, 0) != 0);
        const bool ok = delta == 0;
#pragma unroll
        for (int h = 0; h < NWL; h++) {
            const int w = 32 * h + lane;
            if (w < W) {
                for (int b = 0; b < 32; b++) {
                    const int j = 32 * w + b;
                    if (j < P) {
                        int v = (int)((vp[h] >> b) & 1u) - (int)((vm[h] >> b) & 1u);
                        if (f0neg) v = -v;
                        out[P - 1 - j] = ok ? (int8_t)v : (int8_t)0;
                    }
                }
            }
        }
        return ok;
    }
};

// ---------------------------------------------------------------------------------------------
// R/q divsteps with one CTA of NT threads per element (the root inversions are few and latency
// bound: spreading one chain over 8 warps cuts the per-step critical path ~8x).  Blocked layout:
// thread t holds coefficients t*C .. t*C+C-1 (float-held exact integers, as Divstep).  Per step
// one __syncthreads: each thread publishes its updated g_0 slot (for the shift g <- g/x) and its
// top v slot (for the next v <- x v); thread 0 also publishes the next g_0.  Slots are double
// buffered by step parity.  Coefficients beyond index p are clipped (arrays of p+1, as C15).
// ---------------------------------------------------------------------------------------------
template <class PS, int M, int NT>
struct RqDivstepCTA {
    static constexpr int P = PS::P;
    static constexpr int C = (P + 1 + NT - 1) / NT;
    static constexpr bool ONE_RED = 2LL * ((M + 1) / 2) * ((M + 1) / 2) < (1LL << 24);

    struct Smem {
        float gx[2][NT + 1];     // published g slot 0 (after update), per thread; [NT] = 0
        float vx[2][NT + 1];     // published top v slot, per thread (index t+1; [0] = 0)
        float g1[2];             // thread 0's updated g slot 1 = next g_0
    };

    // gin: this thread's reversed-input slots (g_i = a_{p-1-i}); out: v slots (coefficient
    // p-1-i of the inverse, scaled by f0^-1).  Returns delta == 0 (same value on all threads).
    __device__ static bool invert(float (&g)[C], float (&out)[C], Smem &sm, int t) {
        float f[C], v[C], r[C];
#pragma unroll
        for (int c = 0; c < C; c++) {
            const int i = t * C + c;
            f[c] = (i == 0) ? 1.0f : ((i == P - 1 || i == P) ? -1.0f : 0.0f);
            v[c] = 0.0f;
            r[c] = (i == 0) ? 1.0f : 0.0f;
        }
        if (t == 0) {
            sm.vx[0][0] = 0.0f; sm.vx[1][0] = 0.0f;
            sm.gx[0][NT] = 0.0f; sm.gx[1][NT] = 0.0f;
            sm.g1[1] = g[0];                 // "previous step" publishes the first g_0
        }
        sm.vx[1][t + 1] = 0.0f;
        __syncthreads();
        float g0 = sm.g1[1], f0 = 1.0f;
        int delta = 1;
#pragma unroll 1
        for (int it = 0; it < 2 * P - 1; it++) {
            const int par = it & 1, prv = par ^ 1;
            // v <- x v (neighbour's top slot from the previous step)
            const float vin = sm.vx[prv][t];
#pragma unroll
            for (int c = C - 1; c > 0; c--) v[c] = v[c - 1];
            v[0] = vin;
            if (t * C + C - 1 > P) {
#pragma unroll
                for (int c = 0; c < C; c++)
                    if (t * C + c > P) v[c] = 0.0f;
            }
            const bool swap = (delta > 0) && (g0 != 0.0f);
            delta = swap ? -delta : delta;
            delta += 1;
#pragma unroll
            for (int c = 0; c < C; c++) {
                const float tf = f[c], tv = v[c];
                f[c] = swap ? g[c] : tf;
                g[c] = swap ? tf : g[c];
                v[c] = swap ? r[c] : tv;
                r[c] = swap ? tv : r[c];
            }
            {
                const float tt = f0;
                f0 = swap ? g0 : f0;
                g0 = swap ? tt : g0;
            }
#pragma unroll
            for (int c = 0; c < C; c++) {
                if (ONE_RED) {
                    g[c] = fmodc<M>(__fmaf_rn(f0, g[c], -__fmul_rn(g0, f[c])));
                    r[c] = fmodc<M>(__fmaf_rn(f0, r[c], -__fmul_rn(g0, v[c])));
                } else {
                    g[c] = fmodc<M>(__fmaf_rn(-g0, f[c], fmodc<M>(__fmul_rn(f0, g[c]))));
                    r[c] = fmodc<M>(__fmaf_rn(-g0, v[c], fmodc<M>(__fmul_rn(f0, r[c]))));
                }
            }
            sm.gx[par][t] = g[0];
            sm.vx[par][t + 1] = v[C - 1];
            if (t == 0) sm.g1[par] = (C > 1) ? g[1] : 0.0f;
            __syncthreads();
            // g <- g / x
            const float gin = sm.gx[par][t + 1];
#pragma unroll
            for (int c = 0; c < C - 1; c++) g[c] = g[c + 1];
            g[C - 1] = gin;
            g0 = (C > 1) ? sm.g1[par] : sm.gx[par][1];
        }
        int f0i = (int)f0 % M;
        if (f0i < 0) f0i += M;
        long long s = 1, b = f0i, e = M - 2;                // Fermat: f0^(M-2)
        while (e) { if (e & 1) s = s * b % M; b = b * b % M; e >>= 1; }
#pragma unroll
        for (int c = 0; c < C; c++) out[c] = (float)canon<M>((int)s * (int)v[c]);
        return delta == 0;
    }
};

// One element per CTA of NT threads (all threads of the block call this).
template <class PS, int M, int NT>
__device__ __forceinline__ void inv_row_cta(const InvArgs &a, long long row, int t,
                                            typename RqDivstepCTA<PS, M, NT>::Smem &sm) {
    using DS = RqDivstepCTA<PS, M, NT>;
    constexpr int C = DS::C;
    float g[C], out[C];
#pragma unroll
    for (int c = 0; c < C; c++) {
        const int i = t * C + c;
        g[c] = (i < PS::P) ? (float)load_coef(a.in, row, PS::P - 1 - i) : 0.0f;
    }
    const bool ok = DS::invert(g, out, sm, t);
#pragma unroll
    for (int c = 0; c < C; c++) {
        const int j = t * C + c;
        if (j < PS::P) {
            const int k = PS::P - 1 - j;
            const int val = ok ? (int)out[c] : 0;
            if (a.out_bytes == 2) ((int16_t *)a.out)[row * a.out_stride + k] = (int16_t)val;
            else ((int8_t *)a.out)[row * a.out_stride + k] = (int8_t)val;
        }
    }
    const int ostride = a.out_bytes == 2 ? PS::P8 : PS::P16;
    for (int k = PS::P + t; k < ostride; k += NT) {
        if (a.out_bytes == 2) ((int16_t *)a.out)[row * a.out_stride + k] = 0;
        else ((int8_t *)a.out)[row * a.out_stride + k] = 0;
    }
    if (t == 0 && a.ok) a.ok[row] = ok ? 1 : 0;
}

template <class PS, int M, int NT>
__global__ void __launch_bounds__(NT) divstep_cta_kernel(InvArgs a) {
    __shared__ typename RqDivstepCTA<PS, M, NT>::Smem sm;
    inv_row_cta<PS, M, NT>(a, (long long)blockIdx.x, threadIdx.x, sm);
}

// One element per warp: row `row` of a.in -> a.out, a.ok.
template <class PS, int M>
__device__ __forceinline__ void inv_row_warp(const InvArgs &a, long long row, int lane) {
    const int ostride = a.out_bytes == 2 ? PS::P8 : PS::P16;
    bool ok;
    if constexpr (M == 3) {
        // R/3 rows are int8 (scale 1) on every path that reaches here
        const int8_t *in = (const int8_t *)a.in.ptr + row * a.in.stride;
        int8_t *out = (int8_t *)a.out + row * a.out_stride;
        ok = R3Divstep<PS>::invert(in, out, lane);
    } else {
        using DS = Divstep<PS, M>;
        constexpr int C = DS::C;
        float g[C], out[C];
#pragma unroll
        for (int c = 0; c < C; c++) {
            const int i = lane * C + c;
            g[c] = (i < PS::P) ? (float)load_coef(a.in, row, PS::P - 1 - i) : 0.0f;
        }
        ok = DS::invert(g, out, lane);
#pragma unroll
        for (int c = 0; c < C; c++) {
            const int j = lane * C + c;                     // v index; output coefficient p-1-j
            if (j < PS::P) {
                const int k = PS::P - 1 - j;
                const int val = ok ? (int)out[c] : 0;
                if (a.out_bytes == 2) ((int16_t *)a.out)[row * a.out_stride + k] = (int16_t)val;
                else ((int8_t *)a.out)[row * a.out_stride + k] = (int8_t)val;
            }
        }
    }
    // pad lanes
    for (int k = PS::P + lane; k < ostride; k += 32) {
        if (a.out_bytes == 2) ((int16_t *)a.out)[row * a.out_stride + k] = 0;
        else ((int8_t *)a.out)[row * a.out_stride + k] = 0;
    }
    if (lane == 0 && a.ok) a.ok[row] = ok ? 1 : 0;
}

template <class PS, int M>
__global__ void __launch_bounds__(128) divstep_kernel(InvArgs a) {
    const int lane = threadIdx.x & 31;
    const long long row = (long long)blockIdx.x * 4 + (threadIdx.x >> 5);
    if (row >= a.n) return;
    inv_row_warp<PS, M>(a, row, lane);
}

// Both rings' tree roots in one launch (keygen): blocks [0, nb3) invert R/3 roots, NT/32 per
// block (bitsliced, one warp each); the remaining blocks invert the R/q roots, one per CTA when
// the roots are few (latency bound) or NT/32 per block with one warp each.  The two latency-bound
// chains run side by side instead of one after the other.
template <class PS, int NT>
__global__ void __launch_bounds__(NT) joint_roots_kernel(InvArgs r3, InvArgs rq, int nb3, int rq_cta) {
    __shared__ typename RqDivstepCTA<PS, PS::Q, NT>::Smem sm;
    constexpr int WPB = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if ((int)blockIdx.x < nb3) {
        const long long row = (long long)blockIdx.x * WPB + warp;
        if (row < r3.n) inv_row_warp<PS, 3>(r3, row, lane);
        return;
    }
    const long long b = (long long)blockIdx.x - nb3;
    if (rq_cta) {
        inv_row_cta<PS, PS::Q, NT>(rq, b, threadIdx.x, sm);
    } else {
        const long long row = b * WPB + warp;
        if (row < rq.n) inv_row_warp<PS, PS::Q>(rq, row, lane);
    }
}

// ---------------------------------------------------------------------------------------------
// Keygen repair path: keys of a tree whose R/3 root was not invertible (some g had a factor of
// degree > 64, or the small test was disabled).  Per key (one warp): invert the current g by
// divsteps; while not invertible draw the next attempt (Algorithm 1 line 5 "continue").  Writes
// G, Ginv and attempts for every key of such trees (their tree inverses are meaningless).
// ---------------------------------------------------------------------------------------------
struct RepairArgs {
    uint64_t seed, first, n;
    int B;                       // keys per tree
    const uint8_t *root_ok;      // per tree
    int8_t *G, *Ginv;            // rows of P16
    uint8_t *attempts;
    const uint2 *T;
    const uint32_t *masks;
    int nf;
    int small_check;
    unsigned long long *repaired;
    int *err;
    const int8_t *F;             // rows of P16: f (for u_i = g_i * 3 f_{i^1}); with U
    int16_t *U;                  // rows of P8 or NULL: recompute u_i for repaired keys
};

// u = g * 3 f_sib in R/q for one key (one warp; the rare repair path): folded schoolbook,
// c_k = s_k + s_{k+p} + s_{k+p-1}, s_t = sum_j g_j * 3 f_{t-j}.  f_sib = NULL means 1.
template <class PS>
__device__ void warp_u_product(const int8_t *g, const int8_t *fs, int16_t *u, int lane) {
    constexpr int P = PS::P;
    auto conv = [&](int t) {                          // s_t for t in [0, 2p-2]
        int acc = 0;
        const int j0 = t - (P - 1) > 0 ? t - (P - 1) : 0, j1 = t < P - 1 ? t : P - 1;
        for (int j = j0; j <= j1; j++) acc += (int)g[j] * (int)fs[t - j];
        return 3 * acc;
    };
    for (int k = lane; k < PS::P8; k += 32) {
        int v = 0;
        if (k < P) {
            if (fs) {
                v = conv(k) + conv(k + P) + (k >= 1 ? conv(k + P - 1) : 0);
                v = canon<PS::Q>(v);
            } else {
                v = g[k];
            }
        }
        u[k] = (int16_t)v;
    }
}

template <class PS>
__global__ void __launch_bounds__(128) repair_kernel(RepairArgs a) {
    constexpr int NBL = (PS::NB32 + 31) / 32;
    const int lane = threadIdx.x & 31;
    const uint64_t key_local = (uint64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    if (key_local >= a.n) return;
    if (a.root_ok[key_local / a.B]) return;
    const uint64_t K = sm_at(a.seed, a.first + key_local);
    int8_t *grow = a.G + key_local * PS::P16;
    int8_t *irow = a.Ginv + key_local * PS::P16;
    int attempt = a.attempts ? (int)a.attempts[key_local] - 1 : 0;
    bool ok = false;
    for (int guard = 0; guard < 256; guard++) {
        __syncwarp();
        ok = R3Divstep<PS>::invert(grow, irow, lane);
        if (ok) break;
        // next attempt that passes the small-factor test (if enabled)
        uint32_t pl[NBL], mi[NBL];
        for (;;) {
            ++attempt;
            if (attempt >= 255) break;
            const uint64_t D = sm_at(K, 1 + (uint64_t)attempt);
#pragma unroll
            for (int s = 0; s < NBL; s++) {
                const int b = lane + 32 * s;
                if (b < PS::NB32) small_block<PS>(D, b, pl[s], mi[s]);
                else { pl[s] = 0; mi[s] = 0; }
            }
            if (!a.small_check || small_factor_check<PS, NBL>(pl, mi, a.T, a.masks, a.nf, lane)) break;
        }
        if (attempt >= 255) break;
        __syncwarp();
#pragma unroll
        for (int s = 0; s < NBL; s++) {
            const int b = lane + 32 * s;
            if (32 * b < PS::P16) store_block_int8<PS>(grow, b, pl[s], mi[s]);
        }
        __syncwarp();
    }
    if (!ok) { if (lane == 0) atomicExch(a.err, 2); return; }
    for (int k = PS::P + lane; k < PS::P16; k += 32) irow[k] = 0;
    if (a.U) {
        __syncwarp();
        const uint64_t sib = key_local ^ 1;
        warp_u_product<PS>(grow, sib < a.n ? a.F + sib * PS::P16 : nullptr, a.U + key_local * PS::P8, lane);
    }
    if (lane == 0) {
        if (a.attempts) a.attempts[key_local] = (uint8_t)(attempt + 1);
        atomicAdd(a.repaired, 1ull);
    }
}

}  // namespace sntrup
