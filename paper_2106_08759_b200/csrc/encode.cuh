// encode.cuh -- pk = Rq-encode(h) (radix, C10) and sk = Small-encode(f) ||
// Small-encode(1/g) (C11).  KeyGen step 5: output (h, (f, 1/g)).
//
// Rq-encode merges adjacent pairs (r = R_i + M_i R_{i+1}, m = M_i M_{i+1}), emitting low bytes
// while m >= 2^14, level by level, until one element remains (emitted while m > 1).  The number
// and position of emitted bytes depend only on the moduli M, so the host precomputes a per-level
// table of (M_i, bytes emitted, byte offset) and every pair of a level is processed in parallel.
// One warp per key; the level arrays live in shared memory (values < 2^14 fit uint16).
#pragma once
#include "common.cuh"

namespace sntrup {

constexpr int ENC_MAXLEV = 16;

struct EncTables {
    int nlev;                         // levels with n >= 2
    int lev_n[ENC_MAXLEV];            // elements at the level
    int lev_pair_base[ENC_MAXLEV];    // index of the level's first pair in Mlo/emit/off
    int top_emit, top_off;            // final single element
    const uint32_t *Mlo;              // per pair: M_{2i}
    const uint8_t *emit;              // per pair: bytes emitted
    const uint16_t *off;              // per pair: byte offset of the first emitted byte
    int pk_bytes;
};

struct EncArgs {
    uint64_t n;
    const int16_t *h;      // rows of P8 (may be NULL: no pk)
    const int8_t *f;       // rows of P16 (may be NULL: no sk)
    const int8_t *ginv;    // rows of P16
    uint8_t *pk;           // rows of pk_bytes
    uint8_t *sk;           // rows of 2*SKH
    EncTables t;
};

template <class PS>
__device__ __forceinline__ uint8_t small_byte(const int8_t *row, int j) {
    int v = 0;
#pragma unroll
    for (int t = 0; t < 4; t++) {
        const int i = 4 * j + t;
        if (i < PS::P) v += ((int)row[i] + 1) << (2 * t);
    }
    return (uint8_t)v;
}

template <class PS>
__global__ void __launch_bounds__(128) encode_kernel(EncArgs a) {
    constexpr int WPB = 4;
    __shared__ uint16_t sR[WPB][2][PS::P8];
    __shared__ uint8_t spk[WPB][2112];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint64_t key = (uint64_t)blockIdx.x * WPB + wid;
    if (key >= a.n) return;

    if (a.h) {
        uint16_t *R = sR[wid][0], *R2 = sR[wid][1];
        uint8_t *out = spk[wid];
        const int16_t *hrow = a.h + key * PS::P8;
        for (int i = lane; i < PS::P; i += 32) R[i] = (uint16_t)(hrow[i] + PS::QH);
        __syncwarp();
        for (int lev = 0; lev < a.t.nlev; lev++) {
            const int n = a.t.lev_n[lev];
            const int base = a.t.lev_pair_base[lev];
            for (int i = lane; i < n / 2; i += 32) {
                const uint32_t m0 = a.t.Mlo[base + i];
                uint32_t r = (uint32_t)R[2 * i] + m0 * (uint32_t)R[2 * i + 1];
                const int e = a.t.emit[base + i];
                const int o = a.t.off[base + i];
                for (int t = 0; t < e; t++) { out[o + t] = (uint8_t)(r & 255u); r >>= 8; }
                R2[i] = (uint16_t)r;
            }
            if ((n & 1) && lane == 0) R2[n / 2] = R[n - 1];
            __syncwarp();
            uint16_t *tmp = R; R = R2; R2 = tmp;
        }
        if (lane == 0) {
            uint32_t r = R[0];
            for (int t = 0; t < a.t.top_emit; t++) { out[a.t.top_off + t] = (uint8_t)(r & 255u); r >>= 8; }
        }
        __syncwarp();
        uint8_t *dst = a.pk + key * (uint64_t)a.t.pk_bytes;
        for (int k = lane; k < a.t.pk_bytes; k += 32) dst[k] = out[k];
    }
    if (a.f) {
        uint8_t *dst = a.sk + key * (uint64_t)(2 * PS::SKH);
        const int8_t *frow = a.f + key * PS::P16;
        const int8_t *grow = a.ginv + key * PS::P16;
        for (int j = lane; j < PS::SKH; j += 32) {
            dst[j] = small_byte<PS>(frow, j);
            dst[PS::SKH + j] = small_byte<PS>(grow, j);
        }
    }
}

}  // namespace sntrup
