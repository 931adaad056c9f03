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
    // Per level (host-verified): M_{2i} is the same for every pair of a level (only the last
    // element can be a carried odd one), so every pair but the last emits lev_e bytes at
    // lev_off + lev_e * i; the last pair emits lev_elast bytes.
    uint32_t lev_M[ENC_MAXLEV];
    int lev_e[ENC_MAXLEV], lev_elast[ENC_MAXLEV], lev_off[ENC_MAXLEV];
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

// The same level plan as the host table (C10), evaluated at compile time per parameter set so that
// the kernel's byte-emission loops have constant trip counts (the host checks the two agree).
struct EncPlan {
    int nlev = 0;
    int lev_n[ENC_MAXLEV] = {}, lev_e[ENC_MAXLEV] = {}, lev_elast[ENC_MAXLEV] = {}, lev_off[ENC_MAXLEV] = {};
    uint32_t lev_M[ENC_MAXLEV] = {};
    int top_emit = 0, top_off = 0, pk_bytes = 0;
};

template <int P, int Q>
__host__ __device__ constexpr EncPlan enc_plan() {
    EncPlan t{};
    uint32_t M[P] = {};
    for (int i = 0; i < P; i++) M[i] = (uint32_t)Q;
    int n = P, lev = 0, pos = 0;
    while (n > 1 && lev < ENC_MAXLEV) {
        t.lev_n[lev] = n;
        t.lev_off[lev] = pos;
        t.lev_M[lev] = M[0];
        for (int i = 0; i + 1 < n; i += 2) {
            uint32_t m = M[i] * M[i + 1];
            int e = 0;
            while (m >= 16384u) { e++; m = (m + 255u) >> 8; }
            if (i == 0) t.lev_e[lev] = e;
            t.lev_elast[lev] = e;
            pos += e;
            M[i / 2] = m;                                   // i / 2 <= i: in-place is safe
        }
        if (n & 1) M[n / 2] = M[n - 1];
        n = (n + 1) / 2;
        lev++;
    }
    t.nlev = lev;
    uint32_t m = M[0];
    int e = 0;
    while (m > 1) { e++; m = (m + 255u) >> 8; }
    t.top_emit = e;
    t.top_off = pos;
    t.pk_bytes = pos + e;
    return t;
}

template <class PS>
struct EncPlanOf {
    static constexpr EncPlan v = enc_plan<PS::P, PS::Q>();
};

// level L >= 1 of the radix merge (R -> R2), constant moduli and byte counts
template <class PS, int L>
__device__ __forceinline__ void enc_levels(uint16_t *R, uint16_t *R2, uint8_t *dst, int lane) {
    constexpr EncPlan t = EncPlanOf<PS>::v;
    if constexpr (L < t.nlev) {
        constexpr int n = t.lev_n[L], npairs = n / 2, e = t.lev_e[L], el = t.lev_elast[L], ob = t.lev_off[L];
        constexpr uint32_t m0 = t.lev_M[L];
        for (int i = lane; i < npairs; i += 32) {
            uint32_t r = (uint32_t)R[2 * i] + m0 * (uint32_t)R[2 * i + 1];
            const int o = ob + e * i;
            if (el != e && i == npairs - 1) {
#pragma unroll
                for (int b = 0; b < el; b++) { dst[o + b] = (uint8_t)(r & 255u); r >>= 8; }
            } else {
#pragma unroll
                for (int b = 0; b < e; b++) { dst[o + b] = (uint8_t)(r & 255u); r >>= 8; }
            }
            R2[i] = (uint16_t)r;
        }
        if ((n & 1) && lane == 0) R2[n / 2] = R[n - 1];
        __syncwarp();
        enc_levels<PS, L + 1>(R2, R, dst, lane);
    } else {
        if (lane == 0) {
            uint32_t r = R[0];
#pragma unroll
            for (int b = 0; b < t.top_emit; b++) { dst[t.top_off + b] = (uint8_t)(r & 255u); r >>= 8; }
        }
    }
}

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

// small-encode 4 trits {-1,0,1} packed in a little-endian word -> one byte sum (c+1) 4^t
__device__ __forceinline__ uint32_t small4(uint32_t w) {
    // bytes b_t in {0xff, 0, 1}: ((b_t & 3) + 1) & 3 = c + 1 in {0, 1, 2}, carry-free per byte
    const uint32_t d = ((w & 0x03030303u) + 0x01010101u) & 0x03030303u;
    return (d & 0xffu) | ((d >> 6) & 0x0cu) | ((d >> 12) & 0x30u) | ((d >> 18) & 0xc0u);
}

template <class PS>
__global__ void __launch_bounds__(128) encode_kernel(EncArgs a) {
    constexpr int WPB = 4;
    __shared__ uint16_t sR[WPB][2][PS::P8];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint64_t key = (uint64_t)blockIdx.x * WPB + wid;
    if (key >= a.n) return;

    if (a.h) {
        uint16_t *R = sR[wid][0], *R2 = sR[wid][1];
        uint8_t *dst = a.pk + key * (uint64_t)a.t.pk_bytes;
        const int16_t *hrow = a.h + key * PS::P8;
        // level 0 straight from HBM: 8 coefficients (4 pairs) per lane and 16-byte load; every
        // level-0 pair has M = q*q and emits the same number of bytes e0 at offset e0*i.  Level
        // constants come from the compile-time plan (EncPlanOf, checked against the host table).
        // Emitted bytes go straight to the pk row (consecutive lanes, consecutive bytes).
        {
            constexpr EncPlan pl = EncPlanOf<PS>::v;
            constexpr uint32_t m0 = pl.lev_M[0];
            constexpr int e0 = pl.lev_e[0];
            constexpr int npairs = pl.lev_n[0] / 2;
            static_assert(pl.lev_elast[0] == e0 && pl.nlev >= 2, "level 0: uniform pairs");
            for (int c = lane; c < PS::P8 / 8; c += 32) {
                const uint4 q4 = __ldg(reinterpret_cast<const uint4 *>(hrow) + c);
                const uint32_t w[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
                for (int t = 0; t < 4; t++) {
                    const int i = 4 * c + t;                          // pair index
                    const uint32_t r0 = (uint32_t)((int)(int16_t)(w[t] & 0xffffu) + PS::QH);
                    const uint32_t r1 = (uint32_t)((int)(int16_t)(w[t] >> 16) + PS::QH);
                    if (i < npairs) {
                        uint32_t r = r0 + m0 * r1;
#pragma unroll
                        for (int b = 0; b < e0; b++) { dst[e0 * i + b] = (uint8_t)(r & 255u); r >>= 8; }
                        R2[i] = (uint16_t)r;
                    } else if (2 * i < PS::P) {
                        R2[i] = (uint16_t)r0;                          // odd last element carried
                    }
                }
            }
        }
        __syncwarp();
        enc_levels<PS, 1>(R2, R, dst, lane);
    }
    if (a.f) {
        // 16 trits per 16-byte load -> 4 sk bytes; trits >= P are 0 (pad) and contribute (0+1)
        // in the low-level formula, so the last byte is masked to its P mod 4 coefficients
        uint8_t *dst = a.sk + key * (uint64_t)(2 * PS::SKH);
        const int8_t *rows[2] = {a.f + key * PS::P16, a.ginv + key * PS::P16};
#pragma unroll
        for (int which = 0; which < 2; which++) {
            for (int c = lane; c < PS::P16 / 16; c += 32) {
                const uint4 q4 = __ldg(reinterpret_cast<const uint4 *>(rows[which]) + c);
                const uint32_t w[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
                for (int t = 0; t < 4; t++) {
                    const int j = 4 * c + t;                          // sk byte index
                    if (j < PS::SKH) {
                        uint32_t b = small4(w[t]);
                        const int nvalid = PS::P - 4 * j;             // coefficients present
                        if (nvalid < 4) b &= (1u << (2 * nvalid)) - 1u;
                        dst[which * PS::SKH + j] = (uint8_t)b;
                    }
                }
            }
        }
    }
}

}  // namespace sntrup
