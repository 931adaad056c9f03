// tcxmul.cuh -- "transposed" Hankel form of the int8 tensor-core ring product (one product per
// work item).  Same product as tcmul.cuh (section 3.3, fold x^p = x + 1 folded into
// the second operand, reading Z23), but the GEMM is posed with 16 output coefficients per row:
//
//   c[16 m + n] = sum_k  Bm[m][k] * An[n][k],   Bm[m][k] = bt[16 m + 15 - k],  An[n][k] = a[k + n - 15]
//
// * M side (the MMA's A descriptor): row m' = MB-1-m is the window Z[ZMARG + 16 m' + k] of the
//   reversed folded operand -- a plain VIEW of the staging array Z (rows 16 B apart, K chunks 16 B
//   apart: LBO = 16 B, SBO = 128 B; probed on hardware, scripts/probe/fine_hankel_probe.cu).  No
//   B-row build at all, and with MB = ceil(p/16) <= 64 rows the MMA runs at M = 64: it fetches a
//   64 x 32 B tile (2 KB) per MMA instead of tcmul.cuh's 128 x 32 B Hankel tile (4 KB).
// * N side (the B descriptor): 16 rows per limb of the sliding window of a (16-byte row rho =
//   X[rho .. rho+15], X[x] = a[x - 15]); the limbs' windows are interleaved in blocks of 16 rows so
//   that the LA limbs stack along N (N = 16 LA) under one descriptor (LBO = 256 LA, SBO = 128).
// * Limbs of the Z operand are separate MMA chains (LB accumulator sets of 16 LA columns).
// K = p + 15 (25 K steps of 32 for 761, against 28), so a big x big product is 50 MMAs fetching
// 3 KB each (150 KB) instead of 56 fetching 4.5 KB (252 KB) -- the shared-memory operand fetch is
// what bounds these kernels.
// Thread = accumulator row: it owns 16 consecutive output coefficients (32 contiguous bytes).
// NPR = 2 (the down-sweeps: both children of a parent share the parent's inverse): the shared
// operand u is the window operand -- staged and built once -- and each child is a Z view with its
// own MMA chains, accumulators and mbarrier, so child 0's epilogue overlaps child 1's MMAs.
// The next item is staged (registers -> X / Z staging) while this item's MMAs run; the Z arrays are
// double-buffered by item parity because the MMAs read them directly.
#pragma once
#include "tcmul.cuh"

namespace sntrup {

template <class PS, int LA, int LB, int NPR = 1>
struct TcxGeom {
    static constexpr int P = PS::P;
    static constexpr int MB = (P + 15) / 16;                  // output blocks of 16 = accumulator rows used
    static constexpr int MM = MB <= 64 ? 64 : 128;            // MMA M
    static constexpr int E1 = 16 * MB;
    static constexpr int NKS = (P + 15 + 31) / 32;            // K steps of 32
    static constexpr int K = 32 * NKS;
    static constexpr int NB = 16 * LA;                        // N of the MMA
    static constexpr int WROWS = K + 16;                      // window rows (multiple of 16)
    static constexpr int WBLK = 256 * LA;                     // bytes per block of 16 rows (all limbs)
    static constexpr int W_BYTES = WROWS / 16 * WBLK;
    // X_l (per limb of u): byte 16 + j = limb(a_j); window row r = bytes [r + 1, r + 17)
    static constexpr int HA_LEN = (WROWS + 32 + 127) / 128 * 128;
    static constexpr int PD = P % 8;
    static constexpr int ZMARG = 16;
    static constexpr int ZB_END = ZMARG + E1;                 // b part below, s part from here
    static constexpr int Z_LEN = (ZMARG + 16 * MM + K + 16 + 127) / 128 * 128;
    static constexpr int ZSET = NPR * LB * Z_LEN;             // one parity's Z arrays
    static constexpr int NCHK = PS::P8 / 8;
    static constexpr int CH = (NCHK + 1 + 127) / 128;
    static constexpr int TCU = NPR * LB * NB;
    static constexpr int TCOLS = TCU <= 32 ? 32 : TCU <= 64 ? 64 : 128;
    static constexpr int OFF_W = 0;
    static constexpr int OFF_HA = OFF_W + W_BYTES;
    static constexpr int OFF_ZR = OFF_HA + LA * HA_LEN;
    static constexpr int OFF_BAR = (OFF_ZR + 2 * ZSET + 127) / 128 * 128;
    static constexpr int SMEM = OFF_BAR + 128;
    static constexpr int BY_SMEM = (227 * 1024) / (SMEM + 1024);
    static constexpr int BY_TMEM = 512 / TCOLS;
    static constexpr int MINB = BY_SMEM < BY_TMEM ? (BY_SMEM < 6 ? BY_SMEM : 6) : (BY_TMEM < 6 ? BY_TMEM : 6);
    static_assert(TCU <= 128, "accumulator columns");
    static_assert(16 + PS::P8 <= HA_LEN && WROWS + 17 <= HA_LEN, "X too short");
    static_assert(PD != 0 && NCHK * 8 > P, "p odd: the s-groups need the next chunk");
    static_assert(E1 >= PS::P8, "b part starts inside Z");
    static_assert(ZB_END + P + 8 <= Z_LEN, "Z too short");
    static_assert(W_BYTES % 128 == 0 && HA_LEN % 16 == 0 && Z_LEN % 16 == 0, "alignment");
};

// M = modulus; LA limbs of the window operand u (stacked along N), LB limbs of the Z operands v
// (separate chains); NPR products per item sharing u.  Work items as tcmul.cuh (tc_work).
template <class PS, int M, int LA, int LB, int NPR = 1, bool XOPS = false>
__global__ void __launch_bounds__(128, (TcxGeom<PS, LA, LB, NPR>::MINB)) tcx_mul_kernel(MulArgs a) {
    using G = TcxGeom<PS, LA, LB, NPR>;
    constexpr int P = PS::P, PD = G::PD, CH = G::CH, MM = G::MM;
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *sW = sm + G::OFF_W;
    uint8_t *sHA = sm + G::OFF_HA;
    uint8_t *sZR = sm + G::OFF_ZR;
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + G::OFF_BAR);        // bar[pp]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sm + G::OFF_BAR + 32);
    int *fixs = reinterpret_cast<int *>(sm + G::OFF_BAR + 48);     // D(p-1) hand-off, per product
    int *fixab_s = reinterpret_cast<int *>(sm + G::OFF_BAR + 64);  // a[p-1] b[p-1], [item parity][pp]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    for (int i = tid; i < (G::OFF_BAR - G::OFF_HA) / 16; i += 128)
        reinterpret_cast<uint4 *>(sm + G::OFF_HA)[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    if (tid == 0) {
#pragma unroll
        for (int pp = 0; pp < NPR; pp++) mbar_init(bar + pp, 1);
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
    constexpr uint32_t IDESC = umma_idesc_i8(G::NB, MM);
    uint32_t phase = 0;                                       // mbarrier parity (all products alike)

    uint4 pu[CH], pv[NPR][CH], pn[NPR][CH];
    int pa1 = 0, pb1[NPR];
#pragma unroll
    for (int pp = 0; pp < NPR; pp++) pb1[pp] = 0;
    // window rows 4m+i, stored in the order (i + m/2) mod 4 (8 consecutive threads' 16-byte stores
    // hit 8 distinct bank groups); row r = X bytes [r + 1, r + 17): byte selectors shifted by one
    uint32_t wsel[4];
#pragma unroll
    for (int i = 0; i < 4; i++) wsel[i] = 0x3210u + (uint32_t)(((i + (tid >> 1)) & 3) + 1) * 0x1111u;
    TcWork<NPR> wn;
    auto absent = [&](const TcWork<NPR> &w, int pp) { return pp > 0 && w.orow[pp] < 0; };
    auto prefetch = [&](long long it) {
        if (it >= a.n_out) return;
        tc_work<NPR>(a, it, wn);
        const Opnd du = opnd_or_zero(wn.du, wn.unit_u);
#pragma unroll
        for (int h = 0; h < CH; h++) {
            const int c = tid + 128 * h;
            if (c < G::NCHK) pu[h] = load_chunk(du, c);
            const int cs = c == G::NCHK ? -1 : c;
#pragma unroll
            for (int pp = 0; pp < NPR; pp++) {
                const Opnd dv = opnd_or_zero(wn.dv[pp], wn.unit_v[pp] || absent(wn, pp));
                if (c < G::NCHK) pv[pp][h] = load_chunk(dv, c);
                if (c <= G::NCHK && cs < G::NCHK - 1) pn[pp][h] = load_chunk(dv, cs + 1);
            }
        }
        if (tid == 0) {
            pa1 = load_raw(du, P - 1);
#pragma unroll
            for (int pp = 0; pp < NPR; pp++)
                pb1[pp] = load_raw(opnd_or_zero(wn.dv[pp], wn.unit_v[pp] || absent(wn, pp)), P - 1);
        }
    };
    // ---- stage limbs (registers -> X / Z staging of parity par): as tcmul.cuh
    auto stage = [&](const TcWork<NPR> &w, int par) {
        if (tid == 0) {
            pa1 = coef_fin<XOPS>(w.du, w.unit_u, P - 1, pa1);
#pragma unroll
            for (int pp = 0; pp < NPR; pp++) {
                pb1[pp] = absent(w, pp) ? 0 : coef_fin<XOPS>(w.dv[pp], w.unit_v[pp], P - 1, pb1[pp]);
                fixab_s[par * NPR + pp] = pa1 * pb1[pp];
            }
        }
#pragma unroll
        for (int h = 0; h < CH; h++) {
            const int c = tid + 128 * h;
            if (c < G::NCHK) {
                int uv8[8];
                decode_chunk(pu[h], w.du.bytes, w.du.scale, w.unit_u, c, uv8, XOPS ? w.du.mod3 : 0);
#pragma unroll
                for (int l = 0; l < LA; l++) {
                    int x[8];
#pragma unroll
                    for (int i = 0; i < 8; i++) x[i] = limb_of<LA>(uv8[i], l);
                    SNTRUP_CHECK(16 + 8 * c + 8 <= G::HA_LEN);
                    *reinterpret_cast<uint2 *>(sHA + l * G::HA_LEN + 16 + 8 * c) =
                        make_uint2(pack4(x[0], x[1], x[2], x[3]), pack4(x[4], x[5], x[6], x[7]));
                }
            }
            if (c <= G::NCHK) {
                const int cs = c == G::NCHK ? -1 : c;
#pragma unroll
                for (int pp = 0; pp < NPR; pp++) {
                    uint8_t *zr = sZR + par * G::ZSET + pp * LB * G::Z_LEN;
                    int vv8[8], vn8[8];
                    if (c < G::NCHK)
                        decode_chunk(pv[pp][h], w.dv[pp].bytes, w.dv[pp].scale, w.unit_v[pp], c, vv8,
                                     XOPS ? w.dv[pp].mod3 : 0);
                    else
#pragma unroll
                        for (int i = 0; i < 8; i++) vv8[i] = 0;
                    const bool has_s = cs < G::NCHK - 1;
                    if (has_s) {
                        decode_chunk(pn[pp][h], w.dv[pp].bytes, w.dv[pp].scale, w.unit_v[pp], cs + 1, vn8,
                                     XOPS ? w.dv[pp].mod3 : 0);
                        // s[i] = b[i] + b[i-1] for i = 8cs+PD+j, at Z[ZB_END + p - 1 - i]
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
                        if (c == 0) vv8[0] += pb1[pp];                 // bt[0] = b[0] + b[p-1]
                        const int zo = G::ZB_END - 8 - 8 * c;          // b[8c+i] at ZB_END - 1 - 8c - i
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
    // ---- sliding windows of every limb of u, interleaved in blocks of 16 rows
    auto build = [&]() {
#pragma unroll
        for (int l = 0; l < LA; l++) {
#pragma unroll
            for (int kw = 0; kw < (G::WROWS / 4 + 127) / 128; kw++) {
                const int m = tid + 128 * kw;
                if (m >= G::WROWS / 4) break;
                SNTRUP_CHECK(4 * (m + 5) <= G::HA_LEN);
                const uint32_t *src = reinterpret_cast<const uint32_t *>(sHA + l * G::HA_LEN) + m;
                uint32_t wd[5];
#pragma unroll
                for (int i = 0; i < 5; i++) wd[i] = src[i];
                uint4 *dst = reinterpret_cast<uint4 *>(sW + (m >> 2) * G::WBLK + 256 * l + 64 * (m & 3));
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
        fence_async_smem();
    };
    // ---- MMAs (warp 0, one elected lane): product pp's chains read the Z views of parity par
    auto issue = [&](int par) {
        tc_fence_after();
        const uint64_t bd0 = umma_desc(smem_u32(sW), G::WBLK, 128);
#pragma unroll
        for (int pp = 0; pp < NPR; pp++) {
            const uint32_t z0 = smem_u32(sZR + par * G::ZSET + pp * LB * G::Z_LEN + G::ZMARG);
#pragma unroll 1
            for (int ks = 0; ks < G::NKS; ks++) {
                const uint64_t bd = bd0 + (uint64_t)((ks * 2 * G::WBLK) >> 4);
#pragma unroll
                for (int l = 0; l < LB; l++) {
                    const uint64_t ad = umma_desc(z0 + l * G::Z_LEN + 32 * ks, 16, 128);
                    umma_i8_w(tmem + (pp * LB + l) * G::NB, ad, bd, IDESC, ks > 0 ? 1u : 0u);
                }
            }
            umma_commit_w(bar + pp);
        }
    };
    // accumulator row of this thread (M = 64: rows 16w+i in lanes 32w+i, i < 16)
    const int mrow = MM == 128 ? tid : 16 * warp + lane;
    const bool rowok = (MM == 128 || lane < 16) && mrow < G::MB;
    const int mblk = G::MB - 1 - mrow;                       // output block: coefficients 16 mblk ..
    constexpr int MP1 = (P - 1) / 16, NP1 = (P - 1) % 16;    // D(p-1)
    auto epilogue = [&](int pp, const TcWork<NPR> &w, int par) {
        const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16) + pp * LB * G::NB;
        int v[LB * LA][16];
#pragma unroll
        for (int j = 0; j < LB * LA; j++) tmem_ld16(lane_addr + 16 * j, v[j]);
        tmem_ld_wait();
        // limb recombination, reduced to (-M, M); v[lb * LA + la].  Integer remainders: a float-quotient
        // reduction (I2F / F2I on the conversion pipe, 4 per output) measured 6-10% slower overall
        auto comb = [&](int n) {
            if (LA == 1 && LB == 1) return v[0][n];
            if (LA == 1 || LB == 1) return (64 * v[0][n] + v[1][n]) % M;
            return (4096 * (v[0][n] % M) + 64 * (v[1][n] + v[2][n]) + v[3][n]) % M;
        };
        if (rowok && mblk == MP1) fixs[pp] = comb(NP1);
        // (all threads: the c[0] owner reads the other row's D(p-1))
        __syncthreads();
        const long long orow = w.orow[pp];
        if (!rowok || orow < 0) return;
        int x[16];
#pragma unroll
        for (int n = 0; n < 16; n++) {
            int c = comb(n);
            const int k = 16 * mblk + n;
            if (n == 0 && mblk == 0) c = c - fixs[pp] + fixab_s[par * NPR + pp] % M;
            int vv = k < P ? canon<M>(c) : 0;
            if (XOPS && a.round3) vv -= canon<3>(vv);
            x[n] = vv;
        }
        uint8_t *orp = (pp == 1 && a.out2) ? (uint8_t *)a.out2 + orow * a.out2_stride * a.out_bytes
                                           : (uint8_t *)a.out + orow * a.out_stride * a.out_bytes;
        if (a.out_bytes == 2) {
            int16_t *op = reinterpret_cast<int16_t *>(orp) + 16 * mblk;
            auto pk2 = [](int lo, int hi) { return (uint32_t)(lo & 0xffff) | ((uint32_t)hi << 16); };
            if (16 * mblk < PS::P8)
                reinterpret_cast<uint4 *>(op)[0] = make_uint4(pk2(x[0], x[1]), pk2(x[2], x[3]), pk2(x[4], x[5]), pk2(x[6], x[7]));
            if (16 * mblk + 8 < PS::P8)
                reinterpret_cast<uint4 *>(op)[1] = make_uint4(pk2(x[8], x[9]), pk2(x[10], x[11]), pk2(x[12], x[13]), pk2(x[14], x[15]));
        } else {
            int8_t *op = reinterpret_cast<int8_t *>(orp) + 16 * mblk;
            if (16 * mblk < PS::P16)
                reinterpret_cast<uint4 *>(op)[0] = make_uint4(pack4(x[0], x[1], x[2], x[3]), pack4(x[4], x[5], x[6], x[7]),
                                                              pack4(x[8], x[9], x[10], x[11]), pack4(x[12], x[13], x[14], x[15]));
        }
    };

    // ES: the next item is staged while this item's MMAs run.  Measured (761, isolated): for one
    // product per item the plain loop is faster (big x big 113 vs 103 M/s, big x small 204 vs 174:
    // the second live item costs registers and code), so only the two-product items use it.
    constexpr bool ES = NPR == 2;
    long long it = blockIdx.x;
    if (it < a.n_out) {
        prefetch(it);
        TcWork<NPR> cur = wn;
        int par = 0;
        if constexpr (ES) {
            stage(cur, 0);
            prefetch(it + gridDim.x);
        }
        for (; it < a.n_out; it += gridDim.x) {
            const long long nx = it + gridDim.x;
            if constexpr (!ES) {
                cur = wn;
                stage(cur, par);
            }
            __syncthreads();                              // staging of item `it` complete
            build();
            tc_fence_before();
            __syncthreads();                              // windows built; X staging free
            if (warp == 0) issue(par);
            TcWork<NPR> nxt = cur;
            if constexpr (ES) {
                nxt = wn;
                if (nx < a.n_out) {                       // the next item's limbs while the MMAs run
                    stage(nxt, par ^ 1);
                    prefetch(nx + gridDim.x);
                }
            } else {
                prefetch(nx);
            }
#pragma unroll
            for (int pp = 0; pp < NPR; pp++) {
                if (tid == 0) mbar_wait(bar + pp, phase);
                __syncthreads();
                tc_fence_after();
                epilogue(pp, cur, par);
            }
            phase ^= 1u;
            tc_fence_before();   // TMEM reads ordered before the next item's MMAs (issued after later barriers)
            if constexpr (ES) cur = nxt;
            par ^= 1;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)G::TCOLS));
}

}  // namespace sntrup
