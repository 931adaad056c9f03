// tc4w.cuh -- warp-specialised fp4 ring product with the Hankel A operand in TMEM.
//
// Same product as tc4mul.cuh (the ring product of P:5339-5442 as one Hankel GEMM per product on
// tcgen05.mma kind::mxf4, folded B operand, exact fp32 sums), but the A operand never goes through
// shared memory: the SS form re-reads a 128 x 32-byte A tile from shared memory for every MMA, and
// that fetch -- not the tensor math -- bounded the kernel.  Here one persistent CTA
// per SM (two per SM: 17 warps, 256 TMEM columns each) runs four roles concurrently on a stream of
// work items:
//
//   warps 0-7   A producers: TMEM lane r (= output residue r; warp w owns lanes 32 (w % 4) ..) gets
//               its own Hankel row -- nibbles [1 + r + 64 ks, +64) of the staged digit row hA --
//               built in registers by funnel shifts of 16-byte-aligned loads from five word-shifted
//               copies of hA, and written with tcgen05.st into a ring of NSLOT slots of KG K steps;
//               the two warps of a lane quarter take alternate slots;
//   warps 8-11  loader: raw operand rows arrive by 1D bulk copies (cp.async.bulk) RAW items ahead;
//               item j is staged as digits into hA[j % 2] (the producers' input) and Z, then the
//               folded B rows are built into B[j % 2];
//   warp 16     MMA issuer (converged warp, one elected lane): per slot waits for its A columns,
//               issues tcgen05.mma [acc], [A slot], B descriptor, and commits the slot back to the
//               producers; after the item, commits the B buffer back to the loader and the
//               accumulator to the epilogue;
//   warps 12-15 epilogue: accumulator set j % 2 (double-buffered in TMEM) -> exact reduction mod M,
//               c[0] fix, coalesced stores to HBM; frees the accumulator for item j+2.
//
// All hand-offs are mbarriers in shared memory (producer/consumer phases as in any tcgen05
// pipeline): hfull/hempty (hA buffers), afull/aempty (A slots; aempty is a tcgen05.commit),
// bfull/bempty (B buffers), accfull/accempty (accumulator sets).  Exactness and the operand
// encodings are tc4mul.cuh's (the A/B row construction is shared code).
#pragma once
#include "tc4mul.cuh"

namespace sntrup {

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Wait for an mbarrier phase, suspended in hardware between checks (suspend-time hint ~1 ms) rather
// than polling: many warps of a warp-specialised CTA wait at any time, and polling ones steal issue
// slots and barrier-unit bandwidth from the working ones.  Bounded: a protocol bug traps after
// ~4096 expired hints instead of hanging the GPU.
__device__ __forceinline__ bool mbar_try_wait_sleep(uint64_t *bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase), "r"(1000000u)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void mbar_wait_all(uint64_t *bar, uint32_t phase) {
    int n = 0;
    while (!mbar_try_wait_sleep(bar, phase)) {
        if (++n > (1 << 22)) __trap();
        __nanosleep(64);                 // back off: polling warps steal the working warps' issue slots
    }
}

// Role timing of the warp-specialised kernels (build with -DSNTRUP_WS_TRACE; read with
// sntrup_ws_trace_read): per SM and role, cycles spent waiting on each hand-off and in total.
#ifdef SNTRUP_WS_TRACE
// (trace builds: a wait that times out names itself before trapping)
__device__ __forceinline__ void mbar_wait_dbg(uint64_t *bar, uint32_t phase, int tag) {
    const long long t0 = clock64();
    while (!mbar_try_wait_sleep(bar, phase)) {
        if (clock64() - t0 > (1LL << 30)) {
            printf("tc4w: wait %d timed out (block %d thread %d phase %u)\n", tag, (int)blockIdx.x,
                   (int)threadIdx.x, phase);
            __trap();
        }
    }
}
#define WS_T0() const long long ws_t0_ = clock64()
#define WS_WAIT(slot, bar, ph)                                                         \
    do {                                                                               \
        const long long tw_ = clock64();                                               \
        mbar_wait_dbg(bar, ph, slot);                                                  \
        if (lane == 0 && a.trace) atomicAdd(a.trace + 16 * (blockIdx.x % 160) + (slot), (unsigned long long)(clock64() - tw_)); \
    } while (0)
#define WS_END(slot) \
    if (lane == 0 && a.trace) atomicAdd(a.trace + 16 * (blockIdx.x % 160) + (slot), (unsigned long long)(clock64() - ws_t0_))
#define WS_MARK(v) const long long v = clock64()
#define WS_ADD(slot, v) \
    if (lane == 0 && a.trace) atomicAdd(a.trace + 16 * (blockIdx.x % 160) + (slot), (unsigned long long)(clock64() - v))
#else
#define WS_MARK(v) do {} while (0)
#define WS_ADD(slot, v) do {} while (0)
#define WS_T0() do {} while (0)
#define WS_WAIT(slot, bar, ph) mbar_wait_all(bar, ph)
#define WS_END(slot) do {} while (0)
#endif

template <class PS, int NPR>
struct Tc4wGeom {
    using G = Tc4Geom<PS, 1, NPR, 128>;                       // TA geometry: hA copies, B layout
    static constexpr int KG = 2;                              // K steps per A slot (one tcgen05.st.x16)
    static constexpr int NGRP = (G::NKS + KG - 1) / KG;       // A slot groups per item
    static constexpr int NBUF = 4;                            // items in flight per stage (hA, B, accumulators;
                                                              // the code indexes with j & 3, j >> 2)
    static constexpr int LG = 1;                              // loader groups (4 warps each, alternate items)
    static constexpr int RAWG = 3;                            // raw-row ring slots per loader group
    static constexpr int NPW = 4;                             // producer warps (1 or 2 per TMEM lane quarter)
    static constexpr int CTAS = (G::NB <= 16 && G::NKS <= 20) ? 2 : 1;   // CTAs per SM (512 / CTAS TMEM columns)
    static constexpr int COL_SF = 0;                          // 8 scale-factor columns
    static constexpr int COL_ACC = 32;                        // NBUF accumulator sets of NB columns
    static constexpr int COL_A = (COL_ACC + NBUF * G::NB + 31) / 32 * 32;
    static constexpr int TCOLS = 512 / CTAS;
    static constexpr int NSLOT = ((TCOLS - COL_A) / (8 * KG)) / 2 * 2;   // A ring slots (even)
    // raw operand rows (int8, P16 bytes each): u, then the NPR v rows
    static constexpr int RAW_ROW = PS::P16;
    static constexpr int RAW_SLOT = ((1 + NPR) * RAW_ROW + 127) / 128 * 128;
    // shared memory: B[NBUF] | hA[NBUF] (5 copies each) | Z[LG] | raw rings | barriers
    static constexpr int OFF_B = 0;
    static constexpr int OFF_HA = OFF_B + NBUF * G::B_BYTES;
    static constexpr int OFF_ZR = OFF_HA + NBUF * G::HA_TOTAL;
    static constexpr int ZR_GROUP = (NPR * G::ZR_BYTES + 127) / 128 * 128;
    static constexpr int OFF_RAW = OFF_ZR + LG * ZR_GROUP;
    static constexpr int OFF_BAR = OFF_RAW + LG * RAWG * RAW_SLOT;
    static constexpr int NBAR = 6 * NBUF + 2 * NSLOT + LG * RAWG;
    static constexpr int SMEM = OFF_BAR + NBAR * 8 + 16;
    static constexpr int WARPS = NPW + 4 * LG + 4 + 1;        // producers, loaders, epilogue, MMA
    static constexpr int THREADS = WARPS * 32;
    static_assert(COL_A + 8 * KG * NSLOT <= TCOLS && NSLOT >= NGRP, "TMEM plan");
    static_assert(NBUF == 4, "buffer indexing (j & 3, j >> 2)");
    static_assert((NPW + 4 * LG) % 4 == 0, "epilogue warps start on a lane quarter boundary");
    // the producers read words up to 4 (3 + 2 NKS) + 3 of every hA copy
    static_assert(4 * (4 * (3 + 2 * G::NKS) + 4) <= G::HA_BYTES, "hA copies cover the windows");
    static_assert(G::R0 < 32, "fix row in the first lane quarter");
    static_assert(RAW_ROW % 16 == 0 && G::NCHK * 8 <= RAW_ROW, "raw rows: 16-byte bulk copies");
};

// 1D bulk copy global -> shared, completing on an mbarrier (transaction bytes)
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

// M = modulus (3 or q); one small int8-row operand of each product (LB = 1); NPR products share A.
template <class PS, int M, int NPR>
__global__ void __launch_bounds__(Tc4wGeom<PS, NPR>::THREADS, Tc4wGeom<PS, NPR>::CTAS) tc4w_mul_kernel(MulArgs a) {
    using W = Tc4wGeom<PS, NPR>;
    using G = typename W::G;
    constexpr int P = PS::P;
    constexpr int PD = G::PD;
    constexpr int CH = G::CH;
    constexpr int NKS = G::NKS;
    constexpr int KG = W::KG;
    extern __shared__ __align__(1024) uint8_t sm[];
    constexpr int NBUF = W::NBUF;
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + W::OFF_BAR);
    uint64_t *hfull = bar, *hempty = bar + NBUF, *bfull = bar + 2 * NBUF, *bempty = bar + 3 * NBUF;
    uint64_t *accfull = bar + 4 * NBUF, *accempty = bar + 5 * NBUF;
    uint64_t *afull = bar + 6 * NBUF, *aempty = afull + W::NSLOT;
    uint64_t *rawfull = aempty + W::NSLOT;                          // [LG][RAWG]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sm + W::OFF_BAR + W::NBAR * 8);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    // ---- setup: zero B buffers, hA copies and Z (their pads stay zero forever), barriers, TMEM,
    //      scale factors
    for (int i = tid; i < (W::OFF_RAW - W::OFF_B) / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(sm + W::OFF_B)[i] = make_uint4(0, 0, 0, 0);
    if (tid == 0) {
        for (int i = 0; i < NBUF; i++) {
            mbar_init(hfull + i, 4);
            mbar_init(hempty + i, W::NPW);
            mbar_init(bfull + i, 4);
            mbar_init(bempty + i, 1);
            mbar_init(accfull + i, 1);
            mbar_init(accempty + i, 4);
        }
        for (int i = 0; i < W::NSLOT; i++) {
            mbar_init(afull + i, 4);
            mbar_init(aempty + i, 1);
        }
        for (int i = 0; i < W::LG * W::RAWG; i++) mbar_init(rawfull + i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"((uint32_t)W::TCOLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (warp < 4) {   // scale factors: UE8M0 2^0 in every lane (SFA and SFB both read them)
        const uint32_t la = tmem + ((uint32_t)(warp * 32) << 16) + W::COL_SF;
        const uint32_t s = 0x7f7f7f7fu;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(la),
                     "r"(s), "r"(s), "r"(s), "r"(s), "r"(s), "r"(s), "r"(s), "r"(s));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    const long long first = blockIdx.x, step = gridDim.x;
    const long long nitems = first < a.n_out ? (a.n_out - first + step - 1) / step : 0;

    if (warp < W::NPW) {
        // ================================================================ A producers
        // warp w writes TMEM lanes 32 (w % 4) .. (its lane quarter); the two warps of a quarter take
        // alternate slot groups (KG K steps each) of the item stream.  Lane r: K step ks = nibbles
        // [1 + r + 64 ks, +64) of hA = 8 words funnel-shifted by 4 (r+1 mod 8) bits from words
        // (r+1)/8 + 8 ks .. of copy g (16-byte aligned for the warp)
        constexpr int PSTEP = W::NPW / 4;                           // warps per lane quarter
        const int wq = warp & 3, par = warp >> 2;
        const int r1 = 32 * wq + lane + 1, g = (r1 >> 3) - 4 * wq;   // copy 0..4 of hA
        const uint32_t sh = 4u * (uint32_t)(r1 & 7);
        const uint32_t lane_base = tmem + ((uint32_t)(wq * 32) << 16) + W::COL_A;
        WS_T0();
        int t = par;                                                 // slot-group index within the item stream
        int slot = par, slot_phase = 0;                              // = t % NSLOT, (t / NSLOT) & 1
        for (long long j = 0; j < nitems; j++) {
            const int hb = (int)(j & (NBUF - 1));
            WS_WAIT(0, hfull + hb, (uint32_t)((j >> 2) & 1));
            const uint4 *src = reinterpret_cast<const uint4 *>(sm + W::OFF_HA + hb * G::HA_TOTAL +
                                                               g * G::HA_CSTRIDE) + wq;
            const long long tend = (j + 1) * W::NGRP;
#pragma unroll 1
            for (; t < tend; t += PSTEP) {
                const int k0 = (t - (int)j * W::NGRP) * KG;
                WS_MARK(tc0);
                uint32_t o[8 * KG];
                uint4 q[2 * KG + 1];
#pragma unroll
                for (int i = 0; i < 2 * KG + 1; i++) q[i] = src[2 * k0 + i];
#pragma unroll
                for (int kk = 0; kk < KG; kk++) {
                    const uint32_t x[9] = {q[2 * kk].x, q[2 * kk].y, q[2 * kk].z, q[2 * kk].w,
                                           q[2 * kk + 1].x, q[2 * kk + 1].y, q[2 * kk + 1].z, q[2 * kk + 1].w,
                                           q[2 * kk + 2].x};
#pragma unroll
                    for (int i = 0; i < 8; i++) o[8 * kk + i] = __funnelshift_r(x[i], x[i + 1], sh);
                }
                WS_ADD(13, tc0);
                WS_WAIT(1, aempty + slot, (uint32_t)slot_phase ^ 1u);   // slot free (first use: at once)
                tc_fence_after();
                WS_MARK(tc1);
                const uint32_t ta = lane_base + 8 * KG * slot;
                asm volatile(
                    "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
                    "%15,%16};" ::"r"(ta),
                    "r"(o[0]), "r"(o[1]), "r"(o[2]), "r"(o[3]), "r"(o[4]), "r"(o[5]), "r"(o[6]), "r"(o[7]),
                    "r"(o[8]), "r"(o[9]), "r"(o[10]), "r"(o[11]), "r"(o[12]), "r"(o[13]), "r"(o[14]), "r"(o[15]));
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                WS_ADD(14, tc1);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(afull + slot);
                slot += PSTEP;                                       // (NSLOT even: parity preserved)
                if (slot >= W::NSLOT) { slot -= W::NSLOT; slot_phase ^= 1; }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(hempty + hb);                 // this warp is done with hA[hb]
        }
        WS_END(2);
    } else if (warp < W::NPW + 4 * W::LG) {
        // ================================================================ loader
        // group gi (4 warps) takes items j = gi, gi + LG, ...; raw rows of its k-th item land in its
        // ring slot k % RAWG by 1D bulk copies issued RAWG items ahead by the group's thread 0
        const int gi = (warp - W::NPW) >> 2;
        const int ltid = tid - 32 * (W::NPW + 4 * gi);
        const int bar_id = 1 + gi;
        uint64_t *graw = rawfull + gi * W::RAWG;
        uint8_t *graw_mem = sm + W::OFF_RAW + gi * W::RAWG * W::RAW_SLOT;
        auto issue_raw = [&](long long k) {                          // k-th item of this group
            const long long jj = gi + k * W::LG;
            if (jj >= nitems) return;
            TcWork<NPR> w;
            tc_work<NPR>(a, first + jj * step, w);
            const int rs = (int)(k - (k / W::RAWG) * W::RAWG);
            uint8_t *dst = graw_mem + rs * W::RAW_SLOT;
            uint32_t bytes = 0;
            if (!w.unit_u) bytes += W::RAW_ROW;
#pragma unroll
            for (int pp = 0; pp < NPR; pp++)
                if (!(w.unit_v[pp] || (pp > 0 && w.orow[pp] < 0))) bytes += W::RAW_ROW;
            mbar_expect_tx(graw + rs, bytes);
            if (!w.unit_u) bulk_g2s(dst, w.du.row, W::RAW_ROW, graw + rs);
#pragma unroll
            for (int pp = 0; pp < NPR; pp++)
                if (!(w.unit_v[pp] || (pp > 0 && w.orow[pp] < 0)))
                    bulk_g2s(dst + (1 + pp) * W::RAW_ROW, w.dv[pp].row, W::RAW_ROW, graw + rs);
        };
        if (ltid == 0)
            for (int k = 0; k < W::RAWG; k++) issue_raw(k);
        uint32_t *sZ = reinterpret_cast<uint32_t *>(sm + W::OFF_ZR + gi * W::ZR_GROUP);
        const uint8_t *sZ8 = sm + W::OFF_ZR + gi * W::ZR_GROUP;
        WS_T0();
        int rs = 0, rphase = 0;                                      // raw slot k % RAWG and its phase
        for (long long k = 0;; k++) {
            const long long j = gi + k * W::LG;
            if (j >= nitems) break;
            const int hb = (int)(j & (NBUF - 1));
            TcWork<NPR> w;
            tc_work<NPR>(a, first + j * step, w);
            const uint8_t *raw = graw_mem + rs * W::RAW_SLOT;
            // chunk c of u / v[pp] (8 int8 coefficients as a uint2; zeros for unit / absent rows,
            // whose coefficients come from the unit flags)
            auto rchunk = [&](int row, bool none, bool unit, int c) {
                if (unit) return make_uint2(c == 0 ? 1u : 0u, 0u);          // the unit polynomial
                return none ? make_uint2(0, 0) : reinterpret_cast<const uint2 *>(raw + row * W::RAW_ROW)[c];
            };
            WS_WAIT(3, graw + rs, (uint32_t)rphase);
            // hA buffer hb free (producers finished item j - NBUF)
            WS_WAIT(4, hempty + hb, (uint32_t)(((j >> 2) & 1) ^ 1));
            uint32_t *sHA = reinterpret_cast<uint32_t *>(sm + W::OFF_HA + hb * G::HA_TOTAL);
            int pb1[NPR];
#pragma unroll
            for (int pp = 0; pp < NPR; pp++) {
                const bool none = w.unit_v[pp] || (pp > 0 && w.orow[pp] < 0);
                pb1[pp] = none ? 0 : w.dv[pp].scale * (int)(int8_t)raw[(1 + pp) * W::RAW_ROW + P - 1];
            }
            // ---- stage: digits of u into hA (+ 4 word-shifted copies), folded b into Z
#pragma unroll
            for (int h = 0; h < CH; h++) {
                const int c = ltid + 128 * h;
                if (c < G::NCHK) {
                    const uint2 x = rchunk(0, false, w.unit_u, c);
                    const uint32_t word = e2m1_pack8_int8(x.x, x.y, w.unit_u ? 1 : w.du.scale);
                    SNTRUP_CHECK(4 * (16 + c + 1) <= G::HA_BYTES);
#pragma unroll
                    for (int gg = 0; gg < G::HA_COPIES; gg++) sHA[gg * (G::HA_CSTRIDE / 4) + 16 + c - gg] = word;
                }
                if (c <= G::NCHK) {
                    const int cs = c == G::NCHK ? -1 : c;
#pragma unroll
                    for (int pp = 0; pp < NPR; pp++) {
                        uint32_t *zr = sZ + pp * (G::ZR_BYTES / 4);
                        const int zws = (G::ZB_END + (P - PD) - 8 - 8 * cs) / 8;    // s-group word
                        const int zwb = G::ZB_END / 8 - 1 - c;                      // b[8c+i]
                        const bool unit = w.unit_v[pp];
                        const bool none = !unit && pp > 0 && w.orow[pp] < 0;
                        const int sc = unit ? 1 : w.dv[pp].scale;
                        uint32_t W0 = 0u;
                        if (c < G::NCHK) {
                            const uint2 x = rchunk(1 + pp, none, unit, c);
                            W0 = e2m1_pack8_int8(x.x, x.y, sc);
                        }
                        if (cs < G::NCHK - 1) {
                            const uint2 y = rchunk(1 + pp, none, unit, cs + 1);
                            const uint32_t W1 = e2m1_pack8_int8(y.x, y.y, sc);
                            zr[zws] = nibble_reverse(e2m1_pair_sum(__funnelshift_r(W0, W1, 4 * PD),
                                                                   __funnelshift_r(W0, W1, 4 * (PD - 1)), sc));
                        }
                        if (c < G::NCHK) {
                            uint32_t fw = W0;
                            if (c == 0) {                                    // bt[0] = b[0] + b[p-1]
                                const int b0 = unit ? 1 : none ? 0 : sc * (int)(int8_t)raw[(1 + pp) * W::RAW_ROW];
                                fw = (W0 & ~0xFu) | e2m1_code(b0 + pb1[pp]);
                            }
                            zr[zwb] = nibble_reverse(fw);
                        }
                    }
                }
            }
            asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");   // staged, raw slot read
            if (lane == 0) mbar_arrive(hfull + hb);                  // producers may read hA[hb]
            if (ltid == 0) issue_raw(k + W::RAWG);                   // raw slot rs is free again
            WS_WAIT(5, bempty + hb, (uint32_t)(((j >> 2) & 1) ^ 1));
            // ---- B rows of buffer hb: each Z unit read once, stored into every row window covering it
            uint8_t *sB = sm + W::OFF_B + hb * G::B_BYTES;
#pragma unroll
            for (int h = 0; h < G::UPER; h++) {
                const int wi = ltid + 128 * h;
                if (wi >= G::UITEMS) break;
                const int pl = wi / G::ZUN, u = G::ZU0 + (wi - pl * G::ZUN);     // pl = pp
                const uint4 z = reinterpret_cast<const uint4 *>(sZ8)[pl * (G::ZR_BYTES / 16) + u];
                uint4 *dst = reinterpret_cast<uint4 *>(sB) + pl * G::PCOL;
#pragma unroll
                for (int t = 0; t <= G::NT; t++) {
                    const int c = u - G::zrow(t) / 32;
                    if (c >= 0 && c < G::NCHB) dst[c * G::BLD + t] = z;
                }
            }
            fence_async_smem();
            asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");   // B built; Z free again
            if (lane == 0) mbar_arrive(bfull + hb);
            if (++rs == W::RAWG) { rs = 0; rphase ^= 1; }
        }
        WS_END(6);
    } else if (warp < W::NPW + 4 * W::LG + 4) {
        // ================================================================ epilogue
        const int q = warp & 3;                                      // TMEM lane quarter
        const int r = 32 * q + lane;                                 // accumulator row = residue
        WS_T0();
        for (long long j = 0; j < nitems; j++) {
            const long long it = first + j * step;
            const int ab = (int)(j & (NBUF - 1));
            TcWork<NPR> w;
            tc_work<NPR>(a, it, w);
            int fixab[NPR];
#pragma unroll
            for (int pp = 0; pp < NPR; pp++) fixab[pp] = 0;
            if (r == 0) {                                            // a[p-1] b[p-1] for the c[0] fix
                const int a1 = opnd_coef<false>(w.du, w.unit_u, P - 1);
#pragma unroll
                for (int pp = 0; pp < NPR; pp++)
                    fixab[pp] = (pp > 0 && w.orow[pp] < 0) ? 0 : a1 * opnd_coef<false>(w.dv[pp], w.unit_v[pp], P - 1);
            }
            WS_WAIT(7, accfull + ab, (uint32_t)((j >> 2) & 1));
            tc_fence_after();
            const uint32_t lane_addr = tmem + ((uint32_t)(q * 32) << 16) + W::COL_ACC + ab * G::NB;
            int v[G::NBL][16];
#pragma unroll
            for (int c16 = 0; c16 < G::NBL; c16++) {
                if (16 * c16 + 16 <= G::NB) tmem_ld16(lane_addr + 16 * c16, v[c16]);
                else tmem_ld8(lane_addr + 16 * c16, v[c16]);
            }
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(accempty + ab);               // accumulator set ab free
#pragma unroll
            for (int pp = 0; pp < NPR; pp++) {
                auto comb = [&](int t) {
                    const int col = pp * G::PCOL + t;
                    return __float2int_rn(__int_as_float(v[col >> 4][col & 15]));
                };
                int fix = 0;
                if (q == 0) fix = __shfl_sync(FULL, comb(G::NT), G::R0);   // = D(p-1)
                const long long orow = w.orow[pp];
                if (orow < 0) continue;
                auto store = [&](auto *op) {
                    constexpr int OSTRIDE = sizeof(*op) == 2 ? PS::P8 : PS::P16;
#pragma unroll
                    for (int t = 0; t < G::NT; t++) {
                        const int k = 128 * t + r;
                        if (k >= OSTRIDE) break;
                        int vv;
                        if (k == 0) vv = canon<M>(comb(0) - fix + fixab[pp] % M);
                        else if (M == 3) {
                            const int col = pp * G::PCOL + t;
                            vv = (int)fmodc<3>(__int_as_float(v[col >> 4][col & 15]));   // exact: |D| < 2^20
                        } else vv = canon<M>(comb(t));
                        if (k >= P) vv = 0;
                        op[k] = (std::remove_reference_t<decltype(*op)>)vv;
                    }
                };
                uint8_t *orp = (pp == 1 && a.out2) ? (uint8_t *)a.out2 + orow * a.out2_stride * a.out_bytes
                                                   : (uint8_t *)a.out + orow * a.out_stride * a.out_bytes;
                if (a.out_bytes == 2) store(reinterpret_cast<int16_t *>(orp));
                else store(reinterpret_cast<int8_t *>(orp));
            }
        }
        WS_END(8);
    } else {
        // ================================================================ MMA issuer (last warp,
        // converged; one elected lane issues each MMA / commit)
        constexpr uint32_t IDESC = umma_idesc_mxf4(G::NB);
        uint32_t slot = 0, slot_phase = 0;
        WS_T0();
        for (long long j = 0; j < nitems; j++) {
            const int bb = (int)(j & (NBUF - 1));
            WS_WAIT(9, bfull + bb, (uint32_t)((j >> 2) & 1));
            WS_WAIT(10, accempty + bb, (uint32_t)(((j >> 2) & 1) ^ 1));
            tc_fence_after();
            const uint64_t bd0 = umma_desc(smem_u32(sm + W::OFF_B + bb * G::B_BYTES), G::BLD * 16, 128);
            const uint32_t acc = tmem + W::COL_ACC + bb * G::NB;
            for (int k0 = 0; k0 < NKS; k0 += KG) {
                WS_WAIT(11, afull + slot, slot_phase);
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < KG; kk++) {
                    const int ks = k0 + kk;
                    if (ks < NKS) {
                        const uint64_t bd = bd0 + (uint64_t)((ks * 32 * G::BLD) >> 4);
                        umma_mxf4_ta_w(acc, tmem + W::COL_A + 8 * (KG * slot + kk), bd, IDESC, ks > 0 ? 1u : 0u,
                                     tmem + W::COL_SF);
                    }
                }
                umma_commit_w(aempty + slot);                        // slot free once these MMAs are done
                if (++slot == W::NSLOT) { slot = 0; slot_phase ^= 1u; }
            }
            umma_commit_w(bempty + bb);                              // B buffer free
            umma_commit_w(accfull + bb);                             // accumulator ready
        }
        WS_END(12);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)W::TCOLS));
}

}  // namespace sntrup
