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

// e2m1 code of an integer in [-4, 4]
__device__ __forceinline__ uint32_t e2m1_code(int d) {
    const int a = d < 0 ? -d : d;
    return ((0x65420u >> (4 * a)) & 0xFu) | (d < 0 ? 8u : 0u);
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

// nibble order reversal of a word (nibble i -> nibble 7 - i)
__device__ __forceinline__ uint32_t nibble_reverse(uint32_t x) {
    const uint32_t y = __byte_perm(x, 0, 0x0123);
    return ((y >> 4) & 0x0F0F0F0Fu) | ((y << 4) & 0xF0F0F0F0u);
}

template <class PS, int LB, int NPR>
struct Tc4Geom {
    static constexpr int P = PS::P;
    static constexpr int NKS = (P + 127 + 63) / 64;          // K steps of 64
    static constexpr int K = 64 * NKS;
    static constexpr int NBLK = (2 * P - 1 + 127) / 128;
    static constexpr int NL = (NBLK + 7) / 8 * 8;
    static constexpr int PCOL = (LB * NL + 15) / 16 * 16;
    static constexpr int NB = NPR * PCOL;
    // window rows: the descriptor starts at row 1 and reads rows up to 127 + 32*(2*NKS-1) + 32
    static constexpr int AROWS = 64 * NKS + 128;             // multiple of 8
    static constexpr int A_BYTES = AROWS * 16;
    static constexpr int HA_WORDS = AROWS / 8 + 8;           // 8 nibbles per word; nibble 128 + j = digit(a_j)
    static constexpr int HA_BYTES = (HA_WORDS * 4 + 127) / 128 * 128;
    static constexpr int ZR_BYTES = ((128 * NL + K) / 2 + 127) / 128 * 128;   // nibble 128 NL - 1 - j = digit(b_j)
    static constexpr int NCHB = 2 * NKS;                      // 16-byte K-chunks per B row
    static constexpr int B_BYTES = NCHB * NB * 16;
    static constexpr int RAW_INTS = 128 * NBLK;
    static constexpr int SFCOL = NB;                          // scale-factor columns after the accumulators
    static constexpr int TCOLS_USED = NB + 8;
    static constexpr int TCOLS = TCOLS_USED <= 32 ? 32 : TCOLS_USED <= 64 ? 64 : TCOLS_USED <= 128 ? 128 : 256;
    static constexpr int NCHK = PS::P8 / 8;
    static constexpr int CH = (NCHK + 127) / 128;
    static constexpr int OFF_A = 0;
    static constexpr int OFF_B = OFF_A + A_BYTES;
    static constexpr int OFF_HA = OFF_B + B_BYTES;
    static constexpr int OFF_ZR = OFF_HA + HA_BYTES;
    static constexpr int OFF_BAR = OFF_ZR + NPR * LB * ZR_BYTES;
    static constexpr int SMEM = OFF_BAR + 128;
    static constexpr int BROWS = NPR * LB * NL;
    static constexpr int BITEMS = BROWS * 8;
    static constexpr int BPER = (BITEMS + 127) / 128;
    static_assert(NPR * RAW_INTS * 4 <= A_BYTES, "raw buffers must fit in the A region");
    static_assert(NB <= 256, "N too large");
    static_assert(4 * (16 + NCHK) <= HA_BYTES, "hA too short (staging)");
    static_assert(4 * (AROWS / 8 + 5) <= HA_BYTES, "hA too short (windows)");
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

// M = modulus; A = one digit (the small operand); LB digits for the B operand; NPR products per A.
template <class PS, int M, int LB, int NPR, bool XOPS = false>
__global__ void __launch_bounds__(128) tc4_mul_kernel(MulArgs a) {
    using G = Tc4Geom<PS, LB, NPR>;
    constexpr int P = PS::P;
    constexpr int CH = G::CH;
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *sA = sm + G::OFF_A;
    uint8_t *sB = sm + G::OFF_B;
    uint32_t *sHA = reinterpret_cast<uint32_t *>(sm + G::OFF_HA);
    uint8_t *sZR = sm + G::OFF_ZR;
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + G::OFF_BAR);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sm + G::OFF_BAR + 64);
    int *raw = reinterpret_cast<int *>(sm + G::OFF_A);
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
    int bsrc[G::BPER], bdst[G::BPER], bres[G::BPER];
#pragma unroll
    for (int h = 0; h < G::BPER; h++) {
        const int w = tid + 128 * h;
        if (w < G::BITEMS) {
            const int row = w % G::BROWS, grp = w / G::BROWS;
            const int pl = row / G::NL, t = row - pl * G::NL;       // pl = pp * LB + l
            const int pp = pl / LB, l = pl - pp * LB;
            bres[h] = (grp + row) & 7;
            bsrc[h] = pl * (G::ZR_BYTES / 16) + 4 * (G::NL - 1 - t);
            bdst[h] = pp * G::PCOL + l * G::NL + t;
        } else {
            bsrc[h] = -1; bdst[h] = 0; bres[h] = 0;
        }
    }

    uint4 pu[CH], pv[NPR][CH];
    auto prefetch = [&](long long it) {
        if (it >= a.n_out) return;
        TcWork<NPR> w;
        tc_work<NPR>(a, it, w);
#pragma unroll
        for (int h = 0; h < CH; h++) {
            const int c = tid + 128 * h;
            if (c < G::NCHK) {
                pu[h] = w.unit_u ? make_uint4(0, 0, 0, 0) : load_chunk(w.du, w.ru, c);
#pragma unroll
                for (int pp = 0; pp < NPR; pp++)
                    pv[pp][h] = (w.unit_v[pp] || (pp > 0 && w.orow[pp] < 0)) ? make_uint4(0, 0, 0, 0)
                                                                         : load_chunk(w.dv[pp], w.rv[pp], c);
            }
        }
    };
    prefetch(blockIdx.x);

    for (long long it = blockIdx.x; it < a.n_out; it += gridDim.x) {
        TcWork<NPR> w;
        tc_work<NPR>(a, it, w);
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
                sHA[16 + c] = word;                                  // nibbles 128 + 8c + i
#pragma unroll
                for (int pp = 0; pp < NPR; pp++) {
                    uint32_t dw[LB];
                    if (LB == 1 && w.dv[pp].bytes == 1 && !w.unit_v[pp] && !(XOPS && w.dv[pp].mod3)) {
                        // reversed: coefficient 8c + i -> nibble 7 - i of word 16 NL - 1 - c
                        dw[0] = nibble_reverse(e2m1_pack8_int8(pv[pp][h].x, pv[pp][h].y, w.dv[pp].scale));
                    } else {
                        int vv8[8];
                        decode_chunk(pv[pp][h], w.dv[pp].bytes, w.dv[pp].scale, w.unit_v[pp], c, vv8, XOPS ? w.dv[pp].mod3 : 0);
#pragma unroll
                        for (int l = 0; l < LB; l++) dw[l] = 0;
#pragma unroll
                        for (int i = 0; i < 8; i++) {
                            int v = vv8[i];
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
#pragma unroll
                    for (int l = 0; l < LB; l++)
                        reinterpret_cast<uint32_t *>(sZR + (pp * LB + l) * G::ZR_BYTES)[16 * G::NL - 1 - c] = dw[l];
                }
            }
        }
        __syncthreads();
        // ---- A windows: row rho = nibbles [rho, rho+32); rows 4m..4m+3 share word base m/2
#pragma unroll 1
        for (int m = tid; m < G::AROWS / 4; m += 128) {
            const uint32_t *src = sHA + (m >> 1);
            uint32_t wd[5];
#pragma unroll
            for (int i = 0; i < 5; i++) wd[i] = src[i];
            uint4 *dst = reinterpret_cast<uint4 *>(sA) + 4 * m;
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const int s_ = (i + m) & 3;
                const uint32_t sh = 16u * (uint32_t)(m & 1) + 4u * (uint32_t)s_;
                uint4 o;
                o.x = __funnelshift_r(wd[0], wd[1], sh);
                o.y = __funnelshift_r(wd[1], wd[2], sh);
                o.z = __funnelshift_r(wd[2], wd[3], sh);
                o.w = __funnelshift_r(wd[3], wd[4], sh);
                dst[s_] = o;
            }
        }
        // ---- B rows (aligned 16-byte chunks of the reversed digit arrays)
#pragma unroll
        for (int h = 0; h < G::BPER; h++) {
            if (bsrc[h] < 0) continue;
            const uint4 *src = reinterpret_cast<const uint4 *>(sZR) + bsrc[h];
            uint4 *dst = reinterpret_cast<uint4 *>(sB) + bdst[h];
#pragma unroll 4
            for (int c = bres[h]; c < G::NCHB; c += 8) dst[c * G::NB] = src[c];
        }
        fence_async_smem();
        tc_fence_before();
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
            const uint64_t bd0 = umma_desc(smem_u32(sB), G::NB * 16, 128);
            const uint64_t ad0 = umma_desc(smem_u32(sA) + 16, 512, 128);
#pragma unroll
            for (int ks = 0; ks < G::NKS; ks++) {
                const uint64_t bd = bd0 + (uint64_t)((ks * 32 * G::NB) >> 4);
                const uint64_t ad = ad0 + (uint64_t)((ks * 1024) >> 4);
                umma_mxf4(tmem, ad, bd, IDESC, ks > 0 ? 1u : 0u, tmem + G::SFCOL);
            }
            umma_commit(bar);
        }
        prefetch(it + gridDim.x);
        if (tid == 0) mbar_wait(bar, phase);
        phase ^= 1;
        __syncthreads();
        tc_fence_after();
        const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll
        for (int pp = 0; pp < NPR; pp++) {
            int v[G::PCOL / 16][16];
#pragma unroll
            for (int c16 = 0; c16 < G::PCOL / 16; c16++) tmem_ld16(lane_addr + pp * G::PCOL + 16 * c16, v[c16]);
            tmem_ld_wait();
#pragma unroll
            for (int t = 0; t < G::NBLK; t++) {
                int x = 0;
#pragma unroll
                for (int l = LB - 1; l >= 0; l--) {
                    const int col = l * G::NL + t;
                    x = 9 * x + __float2int_rn(__int_as_float(v[col >> 4][col & 15]));
                }
                raw[pp * G::RAW_INTS + 128 * t + tid] = (LB > 1) ? x % M : x;
            }
        }
        tc_fence_before();
        __syncthreads();
        // (all shared-memory reads of a product issued before its arithmetic: one latency)
        const int ostride_elems = a.out_bytes == 2 ? PS::P8 : PS::P16;
        constexpr int FI = (PS::P16 + 127) / 128;
#pragma unroll
        for (int pp = 0; pp < NPR; pp++) {
            const long long orow = w.orow[pp];
            if (orow < 0) continue;
            const int *rw = raw + pp * G::RAW_INTS;
            int fa[FI], fb[FI], fc[FI];
#pragma unroll
            for (int i = 0; i < FI; i++) {
                const int k = tid + 128 * i;
                fa[i] = fb[i] = fc[i] = 0;
                if (k < P) {
                    fa[i] = rw[k];
                    fb[i] = rw[k + P];
                    fc[i] = k >= 1 ? rw[k + P - 1] : 0;
                }
            }
#pragma unroll
            for (int i = 0; i < FI; i++) {
                const int k = tid + 128 * i;
                if (k >= ostride_elems) break;
                int v = k < P ? canon<M>(fa[i] + fb[i] + fc[i]) : 0;
                if (XOPS && a.round3) v -= canon<3>(v);      // encapsulation's Round
                if (a.out_bytes == 2) ((int16_t *)a.out)[orow * a.out_stride + k] = (int16_t)v;
                else ((int8_t *)a.out)[orow * a.out_stride + k] = (int8_t)v;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)G::TCOLS));
}

}  // namespace sntrup
