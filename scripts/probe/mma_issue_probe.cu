// Probe: why does one thread's tcgen05.mma stream run at ~370 cycles per MMA?  Variants of the
// issue loop (kind::i8, M = 128, N = 32, A in TMEM), one CTA per SM, cycles per MMA per SM.
//   V0: lane 0 of warp 0 alone (diverged warp), per-iteration predicate from a register
//   V1: lane 0 alone, literal enable-input-d, fixed addresses
//   V2: whole warp converged, one lane elected inside the asm (elect.sync)
//   V3: as V2, 4 independent accumulators round robin
//   V4: as V2 but the other warps of the CTA spin on nothing (block of 32 threads)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2106_08759_b200/csrc/tcmul.cuh"
using namespace sntrup;

// V5..V8: kind::mxf4 block-scaled, N = 16, converged warp + elect.sync: V5 A in TMEM, V6 A in
// shared memory, V7 = V5 with warps 1-4 streaming tcgen05.st x16 into other TMEM columns,
// V8 = V5 with 4 accumulators round robin
template <int V>
__global__ void issue(int iters, unsigned long long *cyc) {
    __shared__ __align__(1024) uint8_t sb[128 * 64];
    __shared__ uint64_t bar, ring[4];
    __shared__ uint32_t slot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 128 * 64; i += blockDim.x) sb[i] = (uint8_t)(i * 5);
    if (tid == 0) {
        mbar_init(&bar, 1);
        for (int i = 0; i < 4; i++) mbar_init(&ring[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(256u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const uint64_t bd = umma_desc(smem_u32(sb), (32 / 8) * 128, 128);
    const uint64_t bd16 = umma_desc(smem_u32(sb), (16 / 8) * 128, 128);
    const uint64_t ad = umma_desc(smem_u32(sb), (32 / 8) * 128, 128);   // (A tile: any bytes)
    const uint32_t idf = (1u << 7) | (1u << 10) | ((uint32_t)(16 >> 3) << 17) | (1u << 23) | ((uint32_t)(128 >> 4) << 24);
    if (V >= 5 && warp < 4) {      // scale factors 2^0 at columns 200..207
        const uint32_t s = 0x7f7f7f7fu;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tmem + ((uint32_t)(warp * 32) << 16) + 200),
                     "r"(s), "r"(s), "r"(s), "r"(s), "r"(s), "r"(s), "r"(s), "r"(s));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t idi = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(32 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const unsigned long long t0 = clock64();
    if (V >= 9) {
        // V9: V5 + a commit to mbarrier ring[i/2 % 4] after every 2 MMAs (nobody waits);
        // V10: V9 + tcgen05.fence::after_thread_sync before every pair
        if (warp == 0) {
            for (int i = 0; i < iters; i += 2) {
                if (V == 10) tc_fence_after();
                for (int k = 0; k < 2; k++)
                    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\t"
                                 "@P tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%4], [%4], 1;\n\t}\n"
                                 ::"r"(tmem), "r"(tmem + 128 + 8 * k), "l"(bd16), "r"(idf), "r"(tmem + 200));
                asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\t"
                             "@P tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n"
                             ::"r"(smem_u32(&ring[(i >> 1) & 3])) : "memory");
            }
            asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\t"
                         "@P tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n"
                         ::"r"(smem_u32(&bar)) : "memory");
            mbar_wait(&bar, 0);
        }
    } else if (V >= 5) {
        if (warp == 0) {
            for (int i = 0; i < iters; i++) {
                const uint32_t acc = V == 8 ? tmem + 32 * (i & 3) : tmem;
                if (V == 6)
                    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\t"
                                 "@P tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%4], [%4], 1;\n\t}\n"
                                 ::"r"(acc), "l"(ad), "l"(bd16), "r"(idf), "r"(tmem + 200));
                else
                    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\t"
                                 "@P tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%4], [%4], 1;\n\t}\n"
                                 ::"r"(acc), "r"(tmem + 128), "l"(bd16), "r"(idf), "r"(tmem + 200));
            }
            asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\t"
                         "@P tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n"
                         ::"r"(smem_u32(&bar)) : "memory");
            mbar_wait(&bar, 0);
        } else if (V == 7 && warp <= 4) {
            const uint32_t lr = (uint32_t)(((warp - 1) & 3) * 32) << 16;
            for (int i = 0; i < iters; i++) {
                const uint32_t x = (uint32_t)i;
                asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};"
                             ::"r"(tmem + lr + 160 + 16 * (i & 1)), "r"(x));
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            }
        }
    } else if (V <= 1) {
        if (tid == 0) {
            for (int i = 0; i < iters; i++) {
                if (V == 0) {
                    const uint32_t accum = (i % 56) != 0;
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n"
                                 ::"r"(tmem), "r"(tmem + 128 + 8 * (i & 3)), "l"(bd), "r"(idi), "r"(accum));
                } else {
                    asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, 1;"
                                 ::"r"(tmem), "r"(tmem + 128), "l"(bd), "r"(idi));
                }
            }
            umma_commit(&bar);
            mbar_wait(&bar, 0);
        }
    } else if (warp == 0) {
        for (int i = 0; i < iters; i++) {
            const uint32_t acc = V == 3 ? tmem + 32 * (i & 3) : tmem;
            asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\t"
                         "@P tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, 1;\n\t}\n"
                         ::"r"(acc), "r"(tmem + 128), "l"(bd), "r"(idi));
        }
        asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\t"
                     "@P tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n"
                     ::"r"(smem_u32(&bar)) : "memory");
        mbar_wait(&bar, 0);
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    if (tid == 0) cyc[blockIdx.x] = t1 - t0;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256u));
}

template <int V>
void meas(int threads) {
    const int sms = 148, iters = 4096;
    unsigned long long *d, h[148];
    cudaMalloc(&d, sizeof(h));
    issue<V><<<sms, threads>>>(iters, d);
    issue<V><<<sms, threads>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < sms; i++) mx = mx > h[i] ? mx : (double)h[i];
    printf("V%d threads %3d: %7.1f cycles/MMA (%s)\n", V, threads, mx / iters, cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    meas<0>(128);
    meas<1>(128);
    meas<1>(32);
    meas<2>(128);
    meas<2>(32);
    meas<3>(128);
    meas<5>(128);
    meas<7>(256);
    meas<8>(128);
    meas<6>(128);
    meas<9>(128);
    meas<10>(128);
    return 0;
}
