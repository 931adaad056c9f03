// Probe: tcgen05.mma kind::mxf4.block_scale.block32 with all scale factors = 2^0 (UE8M0 127):
// M=128, N=16 (and 32), K=64 (one MMA) and K=128 (two MMAs), integer digits in [-4, 4] encoded as
// e2m1, no-swizzle K-major core matrices (8 rows x 16 B = 8 x 32 elements, SBO = 128 B between
// row groups, LBO = rows*16 B between 32-element K chunks).  Compares D (fp32) with the host.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../../paper_2106_08759_b200/csrc/tcmul.cuh"
using namespace sntrup;

__host__ __device__ inline uint8_t e2m1(int v) {
    const int a = v < 0 ? -v : v;
    const uint8_t code = a == 0 ? 0 : a == 1 ? 2 : a == 2 ? 4 : a == 3 ? 5 : a == 4 ? 6 : 7;  // 6 -> 7
    return (uint8_t)((v < 0 ? 8 : 0) | code);
}

template <int N, int KS>
__global__ void probe(const int8_t *A, const int8_t *B, float *out) {   // A [128][64*KS], B [N][64*KS]
    constexpr int K = 64 * KS;
    __shared__ __align__(1024) uint8_t sa[128 * K / 2];
    __shared__ __align__(1024) uint8_t sb[N * K / 2];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int tid = threadIdx.x, warp = tid >> 5;
    // byte (row r, byte kb) with kb = k/2: chunk kc = kb/16, x = kb%16
    for (int i = tid; i < 128 * K / 2; i += 128) {
        const int r = i / (K / 2), kb = i % (K / 2);
        const int g = r / 8, j = r % 8, kc = kb / 16, x = kb % 16;
        sa[kc * (128 / 8) * 128 + g * 128 + j * 16 + x] =
            (uint8_t)(e2m1(A[r * K + 2 * kb]) | (e2m1(A[r * K + 2 * kb + 1]) << 4));
    }
    for (int i = tid; i < N * K / 2; i += 128) {
        const int r = i / (K / 2), kb = i % (K / 2);
        const int g = r / 8, j = r % 8, kc = kb / 16, x = kb % 16;
        sb[kc * (N / 8) * 128 + g * 128 + j * 16 + x] =
            (uint8_t)(e2m1(B[r * K + 2 * kb]) | (e2m1(B[r * K + 2 * kb + 1]) << 4));
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
    const uint32_t SFCOL = 64;                       // scale factors at columns 64..71, all 0x7f
    {
        const uint32_t la = tmem + ((uint32_t)(warp * 32) << 16) + SFCOL;
        const uint32_t s = 0x7f7f7f7fu;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(la),
                     "r"(s), "r"(s), "r"(s), "r"(s), "r"(s), "r"(s), "r"(s), "r"(s));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
        tc_fence_after();
        // block-scaled idesc: a/b format E2M1 (MXF4Format = 1), scale format UE8M0, K = 64
        const uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(128 >> 4) << 24);
        for (int ks = 0; ks < KS; ks++) {
            const uint64_t ad = umma_desc(smem_u32(sa) + ks * 2 * (128 / 8) * 128, (128 / 8) * 128, 128);
            const uint64_t bd = umma_desc(smem_u32(sb) + ks * 2 * (N / 8) * 128, (N / 8) * 128, 128);
            const uint32_t acc = ks > 0;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}\n" ::"r"(tmem),
                "l"(ad), "l"(bd), "r"(idesc), "r"(acc), "r"(tmem + SFCOL), "r"(tmem + SFCOL));
        }
        umma_commit(&bar);
    }
    if (tid == 0) mbar_wait(&bar, 0);
    __syncthreads();
    tc_fence_after();
    const uint32_t la = tmem + ((uint32_t)(warp * 32) << 16);
    for (int c = 0; c < N; c++) {
        uint32_t v;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(la + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        out[tid * N + c] = __uint_as_float(v);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128u));
}

template <int N, int KS>
void run() {
    constexpr int K = 64 * KS;
    static int8_t A[128 * K], B[N * K];
    static float ref[128 * N], got[128 * N];
    srand(1234 + N + KS);
    for (int i = 0; i < 128 * K; i++) A[i] = (int8_t)(rand() % 9 - 4);
    for (int i = 0; i < N * K; i++) B[i] = (int8_t)(rand() % 9 - 4);
    for (int r = 0; r < 128; r++)
        for (int n = 0; n < N; n++) {
            int s = 0;
            for (int k = 0; k < K; k++) s += A[r * K + k] * B[n * K + k];
            ref[r * N + n] = (float)s;
        }
    int8_t *dA, *dB; float *dO;
    cudaMalloc(&dA, sizeof(A)); cudaMalloc(&dB, sizeof(B)); cudaMalloc(&dO, sizeof(got));
    cudaMemcpy(dA, A, sizeof(A), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B, sizeof(B), cudaMemcpyHostToDevice);
    probe<N, KS><<<1, 128>>>(dA, dB, dO);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(got, dO, sizeof(got), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < 128 * N; i++) bad += got[i] != ref[i];
    printf("N=%d K=%d: %s, mismatches %d / %d; D[0][0..3] = %g %g %g %g (ref %g %g %g %g)\n", N, K,
           cudaGetErrorString(e), bad, 128 * N, got[0], got[1], got[2], got[3], ref[0], ref[1], ref[2], ref[3]);
    cudaFree(dA); cudaFree(dB); cudaFree(dO);
}

int main() {
    run<16, 1>();
    run<16, 2>();
    run<32, 2>();
    return 0;
}
