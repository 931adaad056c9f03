// common.cuh -- parameter sets, dispatch and small device helpers shared by the sm_100a kernels.
// Product code: shares nothing with oracle/ (DESIGN.md "Boundary").
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

// Bounds checks of shared-memory / global indexing, compiled in only for the checked build
// (_build.build_checked(): -DSNTRUP_BOUNDS_CHECK, libsntrup_gpu_check.so; compute-sanitizer is
// not available on the B200 pool).  A failed check prints and traps.
#ifdef SNTRUP_BOUNDS_CHECK
#include <cstdio>
#define SNTRUP_CHECK(c)                                                                       \
    do {                                                                                      \
        if (!(c)) {                                                                           \
            printf("SNTRUP_CHECK failed: %s (%s:%d) block %d thread %d\n", #c, __FILE__,       \
                   __LINE__, (int)blockIdx.x, (int)threadIdx.x);                               \
            __trap();                                                                         \
        }                                                                                     \
    } while (0)
#else
#define SNTRUP_CHECK(c) \
    do {                \
    } while (0)
#endif

namespace sntrup {

// Parameter sets (p, q, w): 653/761/857 from P:1418-1430 (section 2.1); 953/1013/1277 from
// BASELINE.json configs (reading Z20).  WT = 32-trit words of the small-factor
// residue vector used by the invertibility check (csrc/factor_tables.h, degrees <= 64).
template <int P_, int Q_, int W_, int WT_>
struct Params {
    static constexpr int P = P_;
    static constexpr int Q = Q_;
    static constexpr int W = W_;
    static constexpr int WT = WT_;
    static constexpr int QH = (Q - 1) / 2;
    static constexpr int P8 = (P + 7) / 8 * 8;        // int16 row stride (elements)
    static constexpr int P16 = (P + 15) / 16 * 16;    // int8 row stride (bytes)
    static constexpr int NB32 = (P + 31) / 32;        // 32-coefficient blocks
    static constexpr int NSORT = P <= 1024 ? 1024 : 2048;
    static constexpr int SKH = (P + 3) / 4;           // Small-encode bytes per polynomial
};

using P653 = Params<653, 4621, 288, 2>;
using P761 = Params<761, 4591, 286, 3>;
using P857 = Params<857, 5167, 322, 1>;
using P953 = Params<953, 6343, 396, 2>;
using P1013 = Params<1013, 7177, 448, 5>;
using P1277 = Params<1277, 7879, 492, 1>;

#define SNTRUP_DISPATCH(ps, ...)                                  \
    switch (ps) {                                                 \
    case 653: { using PS = ::sntrup::P653; __VA_ARGS__; } break;  \
    case 761: { using PS = ::sntrup::P761; __VA_ARGS__; } break;  \
    case 857: { using PS = ::sntrup::P857; __VA_ARGS__; } break;  \
    case 953: { using PS = ::sntrup::P953; __VA_ARGS__; } break;  \
    case 1013: { using PS = ::sntrup::P1013; __VA_ARGS__; } break; \
    case 1277: { using PS = ::sntrup::P1277; __VA_ARGS__; } break; \
    default: return SNTRUP_E_PARAM;                               \
    }

constexpr unsigned FULL = 0xffffffffu;

// ---------------------------------------------------------------------------------------------
// C2: SplitMix64 in counter form: SM(s, j) = finaliser(s + (j+1)*gamma).
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t sm_at(uint64_t s, uint64_t j) {
    uint64_t z = s + (j + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// ---------------------------------------------------------------------------------------------
// Bitsliced GF(3): a trit vector of 32 coefficients is a pair of words (pl, mi): bit c of pl
// set <=> coefficient c == +1, bit c of mi set <=> coefficient c == -1.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ void gf3_add(uint32_t &ap, uint32_t &am, uint32_t bp, uint32_t bm) {
    const uint32_t a0 = ~(ap | am), b0 = ~(bp | bm);
    const uint32_t sp = (ap & b0) | (a0 & bp) | (am & bm);
    const uint32_t sm = (am & b0) | (a0 & bm) | (ap & bp);
    ap = sp;
    am = sm;
}

// ---------------------------------------------------------------------------------------------
// Exact centered reduction of float-held integers (|t| < 2^24) modulo M:
// k = round(t / M) via the 1.5*2^23 magic constant, r = t - k*M (single-rounding FMA, exact).
// Result in [-(M+1)/2, (M+1)/2].
// ---------------------------------------------------------------------------------------------
template <int M>
__device__ __forceinline__ float fmodc(float t) {
    constexpr float INV = 1.0f / (float)M;
    const float k = __fadd_rn(__fmaf_rn(t, INV, 12582912.0f), -12582912.0f);
    return __fmaf_rn(-(float)M, k, t);
}

// canonical centered representative of an int in (-2^30, 2^30)
template <int M>
__device__ __forceinline__ int canon(int x) {
    if constexpr (M == 3) {
        if (x > -8192 && x < 8192) {              // multiply-shift remainder (exact on this range)
            const int t = x + 3 * 4096;           // in (4096, 20480): t * 0x5556 / 2^16 - t/3 < 1/3
            const int r = t - 3 * (int)(((unsigned)t * 0x5556u) >> 16);
            return r - 3 * (r >> 1);              // {0, 1, 2} -> {0, 1, -1}
        }
    }
    x %= M;
    if (x > (M - 1) / 2) x -= M;
    if (x < -(M - 1) / 2) x += M;
    return x;
}

template <int M>
__host__ __device__ constexpr int inv_mod_const(int a) {   // a^(M-2) mod M, a in (0, M)
    long long r = 1, b = a, e = M - 2;
    while (e) { if (e & 1) r = r * b % M; b = b * b % M; e >>= 1; }
    return (int)r;
}

// Row descriptor: element (i, k) at ptr + i*stride + k, elements of `bytes` bytes (1 or 2),
// multiplied by `scale` on load.  A NULL ptr means the unit polynomial 1.
// mod3 != 0: each loaded coefficient is reduced to its centered representative mod 3 (an R/q
// element read as an R/3 element, e.g. decapsulation's e mod 3).
struct RowDesc {
    const void *ptr;
    long long stride;   // elements
    int bytes;          // 1 (int8) or 2 (int16)
    int scale;
    int mod3;
};

__device__ __forceinline__ int load_coef(const RowDesc &d, long long row, int k) {
    int v;
    if (d.bytes == 1) v = d.scale * (int)((const int8_t *)d.ptr)[row * d.stride + k];
    else v = d.scale * (int)((const int16_t *)d.ptr)[row * d.stride + k];
    return d.mod3 ? canon<3>(v) : v;
}

}  // namespace sntrup
