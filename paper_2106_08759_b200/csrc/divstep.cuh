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

template <class PS, int M>
__global__ void __launch_bounds__(128) divstep_kernel(InvArgs a) {
    using DS = Divstep<PS, M>;
    constexpr int C = DS::C;
    const int lane = threadIdx.x & 31;
    const long long row = (long long)blockIdx.x * 4 + (threadIdx.x >> 5);
    if (row >= a.n) return;
    float g[C], out[C];
#pragma unroll
    for (int c = 0; c < C; c++) {
        const int i = lane * C + c;
        g[c] = (i < PS::P) ? (float)load_coef(a.in, row, PS::P - 1 - i) : 0.0f;
    }
    const bool ok = DS::invert(g, out, lane);
    const int ostride = a.out_bytes == 2 ? PS::P8 : PS::P16;
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
    // pad lanes
    for (int k = PS::P + lane; k < ostride; k += 32) {
        if (a.out_bytes == 2) ((int16_t *)a.out)[row * a.out_stride + k] = 0;
        else ((int8_t *)a.out)[row * a.out_stride + k] = 0;
    }
    if (lane == 0 && a.ok) a.ok[row] = ok ? 1 : 0;
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
};

template <class PS>
__global__ void __launch_bounds__(128) repair_kernel(RepairArgs a) {
    using DS = Divstep<PS, 3>;
    constexpr int C = DS::C;
    constexpr int NBL = (PS::NB32 + 31) / 32;
    const int lane = threadIdx.x & 31;
    const uint64_t key_local = (uint64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    if (key_local >= a.n) return;
    if (a.root_ok[key_local / a.B]) return;
    const uint64_t K = sm_at(a.seed, a.first + key_local);
    int8_t *grow = a.G + key_local * PS::P16;
    int attempt = a.attempts ? (int)a.attempts[key_local] - 1 : 0;
    float out[C];
    bool ok = false;
    for (int guard = 0; guard < 256; guard++) {
        float g[C];
#pragma unroll
        for (int c = 0; c < C; c++) {
            const int i = lane * C + c;
            g[c] = (i < PS::P) ? (float)grow[PS::P - 1 - i] : 0.0f;
        }
        ok = DS::invert(g, out, lane);
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
#pragma unroll
        for (int s = 0; s < NBL; s++) {
            const int b = lane + 32 * s;
            if (32 * b < PS::P16) store_block_int8<PS>(grow, b, pl[s], mi[s]);
        }
        __syncwarp();
    }
    if (!ok) { if (lane == 0) atomicExch(a.err, 2); return; }
    int8_t *irow = a.Ginv + key_local * PS::P16;
#pragma unroll
    for (int c = 0; c < C; c++) {
        const int j = lane * C + c;
        if (j < PS::P) irow[PS::P - 1 - j] = (int8_t)(int)out[c];
    }
    for (int k = PS::P + lane; k < PS::P16; k += 32) irow[k] = 0;
    if (lane == 0) {
        if (a.attempts) a.attempts[key_local] = (uint8_t)(attempt + 1);
        atomicAdd(a.repaired, 1ull);
    }
}

}  // namespace sntrup
