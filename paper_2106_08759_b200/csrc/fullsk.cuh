// fullsk.cuh -- the full-size secret key (reading Z24).
//
// The paper stores key pairs of 2512 / 2921 / 3321 bytes (App. D):
// pk plus an sk of 3 ceil(p/4) + |pk| + 32 bytes, without naming the extra secret or the hash.
// Ours: sk_full = Small(f) || Small(1/g) || pk || rho || H(pk), rho = ceil(p/4) bytes of the key's
// stream domain DOMAIN_RHO (C2, little-endian words), H(pk) = SHA-512(0x04 || pk)[0..32)
// (FIPS 180-4).  Two kernels: a warp per key copies sk and pk and draws rho (coalesced bytes);
// a thread per key hashes its pk (80 fully unrolled rounds per 128-byte block, 16-word circular
// schedule in registers).
#pragma once
#include "common.cuh"
#include "sha512_k.h"

namespace sntrup {

constexpr uint64_t DOMAIN_RHO = 0x8000000000000000ull;

struct FullSkArgs {
    uint64_t seed, first, n;
    const uint8_t *pk, *sk;
    uint8_t *out;
};

// rows: pk [n][PKB], sk [n][SKB], out [n][SKB + PKB + RB + 32]
template <class PS>
__global__ void __launch_bounds__(128) full_sk_copy_kernel(FullSkArgs a, int pkb, int skb) {
    const int lane = threadIdx.x & 31;
    const uint64_t key = (uint64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    if (key >= a.n) return;
    constexpr int RB = (PS::P + 3) / 4;
    const size_t fsb = (size_t)skb + pkb + RB + 32;
    uint8_t *o = a.out + key * fsb;
    const uint8_t *s = a.sk + key * (size_t)skb, *q = a.pk + key * (size_t)pkb;
    for (int j = lane; j < skb; j += 32) o[j] = s[j];
    for (int j = lane; j < pkb; j += 32) o[skb + j] = q[j];
    const uint64_t D = sm_at(sm_at(a.seed, a.first + key), DOMAIN_RHO);
    for (int j = lane; j < RB; j += 32) o[skb + pkb + j] = (uint8_t)(sm_at(D, (uint64_t)(j / 8)) >> (8 * (j % 8)));
}

__device__ __forceinline__ uint64_t rotr64(uint64_t x, int n) { return (x >> n) | (x << (64 - n)); }

__device__ __forceinline__ void sha512_compress(uint64_t (&H)[8], uint64_t (&W)[16]) {
    uint64_t a = H[0], b = H[1], c = H[2], d = H[3], e = H[4], f = H[5], g = H[6], h = H[7];
#pragma unroll
    for (int t = 0; t < 80; t++) {
        if (t >= 16) {
            const uint64_t w15 = W[(t - 15) & 15], w2 = W[(t - 2) & 15];
            const uint64_t s0 = rotr64(w15, 1) ^ rotr64(w15, 8) ^ (w15 >> 7);
            const uint64_t s1 = rotr64(w2, 19) ^ rotr64(w2, 61) ^ (w2 >> 6);
            W[t & 15] += s1 + W[(t - 7) & 15] + s0;
        }
        const uint64_t S1 = rotr64(e, 14) ^ rotr64(e, 18) ^ rotr64(e, 41);
        const uint64_t T1 = h + S1 + ((e & f) ^ (~e & g)) + SHA512_K[t] + W[t & 15];
        const uint64_t S0 = rotr64(a, 28) ^ rotr64(a, 34) ^ rotr64(a, 39);
        const uint64_t T2 = S0 + ((a & b) ^ (a & c) ^ (b & c));
        h = g; g = f; f = e; e = d + T1; d = c; c = b; b = a; a = T1 + T2;
    }
    H[0] += a; H[1] += b; H[2] += c; H[3] += d; H[4] += e; H[5] += f; H[6] += g; H[7] += h;
}

// H(pk) = SHA-512(0x04 || pk)[0..32) into bytes [SKB + PKB + RB, +32) of each out row
template <class PS>
__global__ void __launch_bounds__(128) sha512_pk_kernel(FullSkArgs a, int pkb, int skb) {
    const uint64_t key = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (key >= a.n) return;
    constexpr int RB = (PS::P + 3) / 4;
    const uint8_t *q = a.pk + key * (size_t)pkb;
    const int L = pkb + 1;                                   // message length in bytes
    const int nblk = (L + 17 + 127) / 128;
    uint64_t H[8];
#pragma unroll
    for (int i = 0; i < 8; i++) H[i] = SHA512_H0[i];
    for (int bk = 0; bk < nblk; bk++) {
        uint64_t W[16];
#pragma unroll
        for (int t = 0; t < 16; t++) {
            uint64_t w = 0;
#pragma unroll
            for (int b = 0; b < 8; b++) {
                const int i = 128 * bk + 8 * t + b;           // message byte index
                uint32_t m;
                if (i == 0) m = 4;
                else if (i < L) m = __ldg(q + i - 1);
                else if (i == L) m = 0x80;
                else m = 0;
                w = (w << 8) | m;
            }
            W[t] = w;
        }
        if (bk == nblk - 1) W[15] = (uint64_t)L * 8;        // 128-bit big-endian length (high half 0)
        sha512_compress(H, W);
    }
    uint8_t *o = a.out + key * ((size_t)skb + pkb + RB + 32) + skb + pkb + RB;
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
        for (int b = 0; b < 8; b++) o[8 * i + b] = (uint8_t)(H[i] >> (56 - 8 * b));
}

}  // namespace sntrup
