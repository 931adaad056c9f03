// Probe: tcgen05.mma kind::mxf4.block_scale.block32 at M = 64 (is it legal, where do the rows
// land in TMEM, is it exact) and the issue-to-completion cycles of a chain of MMAs at M = 64 vs
// M = 128 (N = 16, K = 64 per MMA, no-swizzle K-major operands in shared memory).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../../paper_2106_08759_b200/csrc/tcmul.cuh"
using namespace sntrup;

__host__ __device__ inline uint8_t e2m1(int v) {
    const int a = v < 0 ? -v : v;
    const uint8_t code = a == 0 ? 0 : a == 1 ? 2 : a == 2 ? 4 : a == 3 ? 5 : a == 4 ? 6 : 7;
    return (uint8_t)((v < 0 ? 8 : 0) | code);
}

template <int MM, int N>
__global__ void probe(const int8_t *A, const int8_t *B, float *out, long long *cyc, int reps) {   // A [MM][64], B [N][64]
    constexpr int K = 64;
    __shared__ __align__(1024) uint8_t sa[MM * K / 2];
    __shared__ __align__(1024) uint8_t sb[N * K / 2];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < MM * K / 2; i += 128) {
        const int r = i / (K / 2), kb = i % (K / 2);
        const int g = r / 8, j = r % 8, kc = kb / 16, x = kb % 16;
        sa[kc * (MM / 8) * 128 + g * 128 + j * 16 + x] = (uint8_t)(e2m1(A[r * K + 2 * kb]) | (e2m1(A[r * K + 2 * kb + 1]) << 4));
    }
    for (int i = tid; i < N * K / 2; i += 128) {
        const int r = i / (K / 2), kb = i % (K / 2);
        const int g = r / 8, j = r % 8, kc = kb / 16, x = kb % 16;
        sb[kc * (N / 8) * 128 + g * 128 + j * 16 + x] = (uint8_t)(e2m1(B[r * K + 2 * kb]) | (e2m1(B[r * K + 2 * kb + 1]) << 4));
    }
    if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(128u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t SFCOL = 64;
    {
        const uint32_t la = tmem + ((uint32_t)(warp * 32) << 16) + SFCOL;
        const uint32_t s = 0x7f7f7f7fu;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(la),
                     "r"(s), "r"(s), "r"(s), "r"(s), "r"(s), "r"(s), "r"(s), "r"(s));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    const uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(MM >> 4) << 24);
    const uint64_t ad = umma_desc(smem_u32(sa), (MM / 8) * 128, 128);
    const uint64_t bd = umma_desc(smem_u32(sb), (N / 8) * 128, 128);
    uint32_t ph = 0;
    for (int pass = 0; pass < 2; pass++) {             // pass 0: one MMA (values); pass 1: timing
        const int cnt = pass == 0 ? 1 : reps;
        if (tid == 0) {
            tc_fence_after();
            const long long t0 = clock64();
            for (int i = 0; i < cnt; i++) {
                const uint32_t acc = i > 0;
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}\n" ::"r"(tmem),
                    "l"(ad), "l"(bd), "r"(idesc), "r"(acc), "r"(tmem + SFCOL), "r"(tmem + SFCOL));
            }
            umma_commit(&bar);
            mbar_wait(&bar, ph);
            if (pass == 1) *cyc = clock64() - t0;
        }
        ph ^= 1;
        __syncthreads();
        tc_fence_after();
        if (pass == 0) {
            const uint32_t la = tmem + ((uint32_t)(warp * 32) << 16);
            for (int c = 0; c < N; c++) {
                uint32_t v;
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(la + c));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                out[tid * N + c] = __uint_as_float(v);        // by TMEM lane
            }
        }
        tc_fence_before();
        __syncthreads();
    }
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128u));
}

template <int MM, int N>
void run(int reps) {
    constexpr int K = 64;
    static int8_t A[MM * K], B[N * K];
    static float ref[MM * N], got[128 * N];
    srand(99 + MM + N);
    for (int i = 0; i < MM * K; i++) A[i] = (int8_t)(rand() % 9 - 4);
    for (int i = 0; i < N * K; i++) B[i] = (int8_t)(rand() % 9 - 4);
    for (int r = 0; r < MM; r++)
        for (int n = 0; n < N; n++) {
            int s = 0;
            for (int k = 0; k < K; k++) s += A[r * K + k] * B[n * K + k];
            ref[r * N + n] = (float)s;
        }
    int8_t *dA, *dB; float *dO; long long *dc;
    cudaMalloc(&dA, sizeof(A)); cudaMalloc(&dB, sizeof(B)); cudaMalloc(&dO, sizeof(got)); cudaMalloc(&dc, 8);
    cudaMemcpy(dA, A, sizeof(A), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B, sizeof(B), cudaMemcpyHostToDevice);
    cudaMemset(dO, 0, sizeof(got));
    probe<MM, N><<<1, 128>>>(dA, dB, dO, dc, reps);
    cudaError_t e = cudaDeviceSynchronize();
    long long cyc = 0;
    cudaMemcpy(got, dO, sizeof(got), cudaMemcpyDeviceToHost);
    cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    // layouts: M=128 row r in lane r; M=64 try lane 32(r/16) + r%16 and lane r
    int bad_a = 0, bad_b = 0;
    for (int r = 0; r < MM; r++)
        for (int n = 0; n < N; n++) {
            const int la = MM == 128 ? r : 32 * (r / 16) + r % 16;
            bad_a += got[la * N + n] != ref[r * N + n];
            bad_b += got[r * N + n] != ref[r * N + n];
        }
    printf("M=%d N=%d: %s; mismatches (lane 32(r/16)+r%%16 layout) %d, (lane r) %d of %d; %d MMAs in %lld cycles = %.1f cyc/MMA\n",
           MM, N, cudaGetErrorString(e), bad_a, bad_b, MM * N, reps, cyc, (double)cyc / reps);
    cudaFree(dA); cudaFree(dB); cudaFree(dO); cudaFree(dc);
}

int main() {
    run<128, 16>(2000);
    run<64, 16>(2000);
    run<128, 32>(2000);
    run<64, 32>(2000);
    return 0;
}
