// ringmul.cuh -- batched ring products in R/q and R/3 (v1: register-tiled schoolbook on the
// integer pipes).
//
// The product of section 3.3: full product of two length-p polynomials, then
// reduction by x^p - x - 1 (x^p = x + 1), coefficients centered mod q (or mod 3).  One CTA per
// product; thread t owns two 8-coefficient output tiles (t and its mirror) so every thread does
// ~p/8 + 2 inner 8x8 blocks (balanced triangle).  Accumulation is int32 with a periodic
// reduction when both operands are full-size (|a_i b_j| <= ((q-1)/2)^2).
//
// Modes (how a CTA finds its operands; the tree levels of batchInv):
//   ZIP   : out[i] = X[i] * Y[i]
//   PAIRS : out[j] = X[2j] * X[2j+1]          (up-sweep; X[2j] alone if 2j+1 >= cnt_in)
//   DOWN  : out[i] = Y[i>>1] * X[i^1]         (down-sweep; Y[i>>1] alone if i^1 >= cnt_in)
//   DOWN2 : DOWN with both children of parent j in one work item (n_out = parents; tensor path)
//   SIB   : out[i] = X[i] * Y[i^1]            (Y[i^1] = 1 if i^1 >= cnt_in)
//   DOWNH : out[i] = Y[i>>1] * X[i]           (no sibling swap)
//   DOWNH2: DOWNH with both children of parent j in one work item (tensor path)
#pragma once
#include "common.cuh"

namespace sntrup {

enum MulMode { MUL_ZIP = 0, MUL_PAIRS = 1, MUL_DOWN = 2, MUL_DOWN2 = 3, MUL_SIB = 4, MUL_DOWNH = 5, MUL_DOWNH2 = 6,
               MUL_UP0 = 7, MUL_ODDSIB = 8 };
// (tensor paths only)
//   UP0   : item j, A = Y[2j+1] (unit if absent): out[2j] = X[2j] * A and out2[j] = Y[2j] * A
//           (keygen: u_{2j} = g_{2j} * 3f_{2j+1} and the R/q tree's level 1, 3f_{2j} * 3f_{2j+1},
//           share 3f_{2j+1})
//   ODDSIB: out[2j+1] = X[2j+1] * Y[2j]   (the remaining u_{2j+1})

struct MulArgs {
    int mode;
    long long n_out;
    long long cnt_in;
    RowDesc X, Y;
    void *out;
    long long out_stride;   // elements
    int out_bytes;          // 1 or 2
    int periodic;           // both operands full-size -> lazy reductions inside the tile loop
    int swap;               // tensor-core path: the second operand takes the A (Hankel) role
    int round3;             // post-op: each output coefficient to the nearest multiple of 3
    void *out2;             // MUL_UP0: second product's output rows (stride out2_stride)
    long long out2_stride;
    unsigned long long *trace;   // SNTRUP_WS_TRACE builds: role timing of the warp-specialised kernels
};

template <int NP>
struct MulSmem {
    int a[NP];
    int b[24 + NP + 8];     // b[-24 .. NP+8) zero-padded window source
    int raw[2 * NP];
};

template <int M, int NP>
__device__ __forceinline__ void mul_tile(const int *__restrict__ sa, const int *__restrict__ sbp,
                                         int *__restrict__ raw, int k0, bool periodic) {
    // acc[r] = sum_i a_i * b_{k0 + r - i}, i over the aligned 8-blocks that can contribute
    constexpr int QH = (M - 1) / 2;
    constexpr long long TERM = (long long)QH * QH;
    constexpr int RB = (int)((2147483647LL - 4194304LL) / (8 * TERM) > 1000000
                                 ? 1000000 : (2147483647LL - 4194304LL) / (8 * TERM));
    const int lo = max(0, k0 - NP + 1) & ~7;
    const int hi = min(NP - 1, k0 + 7) & ~7;
    int acc[8];
#pragma unroll
    for (int r = 0; r < 8; r++) acc[r] = 0;
    int d = k0 - lo;                                   // multiple of 8
    int wl[8], wh[8];
    {
        const int4 *p0 = reinterpret_cast<const int4 *>(sbp + d);
        const int4 *p1 = reinterpret_cast<const int4 *>(sbp + d - 8);
        int4 x0 = p0[0], x1 = p0[1], y0 = p1[0], y1 = p1[1];
        wh[0] = x0.x; wh[1] = x0.y; wh[2] = x0.z; wh[3] = x0.w;
        wh[4] = x1.x; wh[5] = x1.y; wh[6] = x1.z; wh[7] = x1.w;
        wl[0] = y0.x; wl[1] = y0.y; wl[2] = y0.z; wl[3] = y0.w;
        wl[4] = y1.x; wl[5] = y1.y; wl[6] = y1.z; wl[7] = y1.w;
    }
    int cnt = 0;
    for (int i0 = lo; i0 <= hi; i0 += 8) {
        const int4 *pa = reinterpret_cast<const int4 *>(sa + i0);
        const int4 a0 = pa[0], a1 = pa[1];
        const int av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        // prefetch the next low window while multiplying
        const int4 *pn = reinterpret_cast<const int4 *>(sbp + d - 16);
        const int4 n0 = pn[0], n1 = pn[1];
#pragma unroll
        for (int s = 0; s < 8; s++)
#pragma unroll
            for (int r = 0; r < 8; r++) {
                const int idx = 8 + r - s;             // 1 .. 15 : b[d - 8 + idx]
                const int bv = idx < 8 ? wl[idx] : wh[idx - 8];
                acc[r] += av[s] * bv;
            }
#pragma unroll
        for (int u = 0; u < 8; u++) wh[u] = wl[u];
        wl[0] = n0.x; wl[1] = n0.y; wl[2] = n0.z; wl[3] = n0.w;
        wl[4] = n1.x; wl[5] = n1.y; wl[6] = n1.z; wl[7] = n1.w;
        d -= 8;
        if (periodic && ++cnt == RB) {
            cnt = 0;
#pragma unroll
            for (int r = 0; r < 8; r++) acc[r] %= M;
        }
    }
#pragma unroll
    for (int r = 0; r < 8; r++) raw[k0 + r] = acc[r] % M;
}

template <class PS, int M>
__global__ void __launch_bounds__((PS::P8 / 8 + 31) / 32 * 32) ring_mul_kernel(MulArgs a) {
    constexpr int NP = PS::P8;
    constexpr int T = NP / 8;                          // tiles per half = working threads
    __shared__ __align__(16) MulSmem<NP> sm;
    const int tid = threadIdx.x;
    int *sb = sm.b + 24;

    for (long long prod = blockIdx.x; prod < a.n_out; prod += gridDim.x) {
        long long ra, rb;
        const RowDesc *da, *db;
        bool unit_b = false;
        if (a.mode == MUL_ZIP) {
            da = &a.X; ra = prod; db = &a.Y; rb = prod;
        } else if (a.mode == MUL_PAIRS) {
            da = &a.X; ra = 2 * prod; db = &a.X; rb = 2 * prod + 1;
            unit_b = rb >= a.cnt_in;
        } else if (a.mode == MUL_SIB) {
            da = &a.X; ra = prod; db = &a.Y; rb = prod ^ 1;
            unit_b = rb >= a.cnt_in;
        } else if (a.mode == MUL_DOWNH) {
            da = &a.Y; ra = prod >> 1; db = &a.X; rb = prod;
        } else {
            da = &a.Y; ra = prod >> 1; db = &a.X; rb = prod ^ 1;
            unit_b = rb >= a.cnt_in;
        }
        __syncthreads();                               // smem reuse across grid-stride iterations
        for (int k = tid; k < NP; k += blockDim.x) {
            sm.a[k] = k < PS::P ? load_coef(*da, ra, k) : 0;
            sb[k] = unit_b ? (k == 0) : (k < PS::P ? load_coef(*db, rb, k) : 0);
        }
        for (int k = tid; k < 24; k += blockDim.x) sm.b[k] = 0;
        for (int k = tid; k < 8; k += blockDim.x) sb[NP + k] = 0;
        __syncthreads();
        if (tid < T) {
            mul_tile<M, NP>(sm.a, sb, sm.raw, 8 * tid, a.periodic != 0);
            mul_tile<M, NP>(sm.a, sb, sm.raw, 2 * NP - 8 - 8 * tid, a.periodic != 0);
        }
        __syncthreads();
        // fold with x^p = x + 1: c_k = raw_k + raw_{k+p} + raw_{k+p-1} (k >= 1), then center
        const int ostride_elems = a.out_bytes == 2 ? PS::P8 : PS::P16;
        for (int k = tid; k < ostride_elems; k += blockDim.x) {
            int v = 0;
            if (k < PS::P) {
                v = sm.raw[k] + sm.raw[k + PS::P] + (k >= 1 ? sm.raw[k + PS::P - 1] : 0);
                v = canon<M>(v);
                if (a.round3) v -= canon<3>(v);
            }
            if (a.out_bytes == 2) ((int16_t *)a.out)[prod * a.out_stride + k] = (int16_t)v;
            else ((int8_t *)a.out)[prod * a.out_stride + k] = (int8_t)v;
        }
    }
}

}  // namespace sntrup
