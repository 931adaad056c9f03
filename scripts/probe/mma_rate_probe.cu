// Probe: tcgen05.mma issue / throughput rates on B200 for the ring-product shapes (M = 128,
// N = 16 / 32, kind::mxf4 K = 64 and kind::i8 K = 32), A from shared memory (SS) or TMEM (TS):
// how many cycles per MMA per SM with 1, 2 or 4 issuing warps per CTA, 1 or 2 CTAs per SM, a
// commit + mbarrier wait every G MMAs (a work item), and concurrent tcgen05.st traffic (the A
// producers of the warp-specialised kernel).  Not product code: measurements for DESIGN.md 6.1.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_rate_probe mma_rate_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2106_08759_b200/csrc/tcmul.cuh"
using namespace sntrup;

// KIND 0 = mxf4 (block-scaled, K 64), 1 = i8 (K 32); TS = A from TMEM
template <int KIND, bool TS, int N>
__global__ void __launch_bounds__(256) rate(int iters, int nis, int group, int sttm, int tcols,
                                            unsigned long long *cyc) {
    __shared__ __align__(1024) uint8_t sa[128 * 32];
    __shared__ __align__(1024) uint8_t sb[256 * 32];
    __shared__ uint64_t bar[4];
    __shared__ uint32_t slot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 128 * 32; i += 256) sa[i] = (uint8_t)(i * 7);
    for (int i = tid; i < 256 * 32; i += 256) sb[i] = (uint8_t)(i * 5);
    if (tid == 0) {
        for (int i = 0; i < 4; i++) mbar_init(&bar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"((uint32_t)tcols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    // columns: [0, 8) scale factors, accumulators from 32, A at tcols - 64 (32 cols), stores at tcols - 32
    const uint32_t lrow = (uint32_t)((warp & 3) * 32) << 16;
    if (warp < 4) {
        const uint32_t s = 0x7f7f7f7fu;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tmem + lrow),
                     "r"(s), "r"(s), "r"(s), "r"(s), "r"(s), "r"(s), "r"(s), "r"(s));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const unsigned long long t0 = clock64();
    if (warp < nis && lane == 0) {
        const uint64_t ad = umma_desc(smem_u32(sa), (128 / 8) * 128, 128);
        const uint64_t bd = umma_desc(smem_u32(sb), (N / 8) * 128, 128);
        const uint32_t idf = (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(128 >> 4) << 24);
        const uint32_t idi = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint32_t acc = tmem + 32 + (N > 32 ? N : 32) * warp;
        uint32_t ph = 0;
        for (int i = 0; i < iters; i++) {
            const uint32_t accum = (i % group) != 0;
            const uint32_t ta = tmem + (tcols - 64) + 8 * (i & 3);
            if (KIND == 0 && !TS)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%5], p;\n\t}\n"
                             ::"r"(acc), "l"(ad), "l"(bd), "r"(idf), "r"(accum), "r"(tmem));
            if (KIND == 0 && TS)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%5], [%5], p;\n\t}\n"
                             ::"r"(acc), "r"(ta), "l"(bd), "r"(idf), "r"(accum), "r"(tmem));
            if (KIND == 1 && !TS)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
                             ::"r"(acc), "l"(ad), "l"(bd), "r"(idi), "r"(accum));
            if (KIND == 1 && TS)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n"
                             ::"r"(acc), "r"(ta), "l"(bd), "r"(idi), "r"(accum));
            if ((i + 1) % group == 0) {
                umma_commit(&bar[warp]);
                mbar_wait(&bar[warp], ph);
                ph ^= 1;
            }
        }
        umma_commit(&bar[warp]);
        mbar_wait(&bar[warp], ph);
    } else if (warp >= 4 && sttm) {
        // A-producer-like traffic: 32-column stores into columns 224 .. 224 + 32 (not read by MMAs)
        for (int i = 0; i < sttm; i++) {
            const uint32_t x = (uint32_t)i;
            asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
                         "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(tmem + lrow + tcols - 32), "r"(x));
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    if (tid == 0) cyc[blockIdx.x] = t1 - t0;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)tcols));
}

template <int KIND, bool TS, int N>
void meas(const char *name, int ctas_per_sm, int nis, int group, int sttm) {
    const int sms = 148, iters = 14 * 200;
    unsigned long long *d, h[2 * 148];
    cudaMalloc(&d, sizeof(h));
    const int tcols = ctas_per_sm == 1 ? 512 : 256;
    rate<KIND, TS, N><<<sms * ctas_per_sm, 256>>>(iters, nis, group, sttm ? iters * 2 : 0, tcols, d);
    rate<KIND, TS, N><<<sms * ctas_per_sm, 256>>>(iters, nis, group, sttm ? iters * 2 : 0, tcols, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(unsigned long long) * sms * ctas_per_sm, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < sms * ctas_per_sm; i++) mx = mx > h[i] ? mx : (double)h[i];
    const double mmas_per_sm = (double)iters * nis * ctas_per_sm;
    printf("%-6s %s N=%3d  ctas/SM %d  issuers %d  group %4d  sttm %d : %7.1f cycles/MMA/SM  (%s)\n", name,
           TS ? "TS" : "SS", N, ctas_per_sm, nis, group, sttm, mx / mmas_per_sm, cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    for (int g : {1000000, 14, 4}) {
        meas<0, true, 16>("mxf4", 1, 1, g, 0);
        meas<0, false, 16>("mxf4", 1, 1, g, 0);
    }
    meas<0, true, 16>("mxf4", 1, 2, 14, 0);
    meas<0, true, 16>("mxf4", 1, 4, 14, 0);
    meas<0, true, 16>("mxf4", 2, 1, 14, 0);
    meas<0, true, 16>("mxf4", 2, 2, 14, 0);
    meas<0, true, 16>("mxf4", 1, 1, 14, 1);
    meas<0, true, 16>("mxf4", 1, 4, 14, 1);
    meas<0, false, 16>("mxf4", 1, 4, 14, 0);
    meas<0, true, 32>("mxf4", 1, 1, 14, 0);
    meas<0, true, 32>("mxf4", 1, 4, 14, 0);
    meas<1, true, 32>("i8", 1, 1, 56, 0);
    meas<1, true, 32>("i8", 1, 2, 56, 0);
    meas<1, true, 32>("i8", 1, 4, 56, 0);
    meas<1, false, 32>("i8", 1, 1, 56, 0);
    meas<1, false, 32>("i8", 1, 4, 56, 0);
    meas<1, true, 32>("i8", 1, 4, 56, 1);
    meas<1, true, 64>("i8", 1, 4, 56, 0);
    meas<1, true, 16>("i8", 1, 4, 56, 0);
    meas<1, true, 128>("i8", 1, 1, 56, 0);
    meas<1, true, 128>("i8", 1, 2, 56, 0);
    return 0;
}
