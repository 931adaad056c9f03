// Probe: where does tcgen05.mma kind::i8 with M=64 (cta_group::1) place D[r][n] in TMEM?
// A[r][k] = (k == 0) ? r + 1 : 0 (64 x 32, K-major no-swizzle), B[n][k] = (k == 0) ? n + 1 : 0
// (N x 32) -> D[r][n] = (r+1)(n+1).  Dumps all 128 lanes x N columns.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2106_08759_b200/csrc/tcmul.cuh"
using namespace sntrup;

template <int MM, int N>
__global__ void probe(int *out) {
    __shared__ __align__(1024) uint8_t sa[MM * 32];
    __shared__ __align__(1024) uint8_t sb[N * 32];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int tid = threadIdx.x, warp = tid >> 5;
    // K-major no-swizzle core matrices: (row group g, k-chunk kc) at g*128 + kc*LBO; row j at +16j
    for (int i = tid; i < MM * 32; i += 128) {
        const int r = i / 32, k = i % 32;
        const int g = r / 8, j = r % 8, kc = k / 16, x = k % 16;
        sa[g * 128 + kc * (MM / 8) * 128 + j * 16 + x] = (k == 0) ? (uint8_t)(r + 1) : 0;
    }
    for (int i = tid; i < N * 32; i += 128) {
        const int r = i / 32, k = i % 32;
        const int g = r / 8, j = r % 8, kc = k / 16, x = k % 16;
        sb[g * 128 + kc * (N / 8) * 128 + j * 16 + x] = (k == 0) ? (uint8_t)(r + 1) : 0;
    }
    if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(256u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    // zero TMEM region first via a dummy: store zeros
    {
        const uint32_t la = tmem + ((uint32_t)(warp * 32) << 16);
        for (int c = 0; c < 256; c++) asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(la + c), "r"(0));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
        tc_fence_after();
        const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(MM >> 4) << 24);
        const uint64_t ad = umma_desc(smem_u32(sa), (MM / 8) * 128, 128);
        const uint64_t bd = umma_desc(smem_u32(sb), (N / 8) * 128, 128);
        umma_i8(tmem, ad, bd, idesc, 0u);
        umma_commit(&bar);
    }
    if (tid == 0) mbar_wait(&bar, 0);
    __syncthreads();
    tc_fence_after();
    const uint32_t la = tmem + ((uint32_t)(warp * 32) << 16);
    for (int c = 0; c < 2 * N; c++) {
        int v;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(la + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        out[tid * 2 * N + c] = v;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256u));
}

template <int MM, int N>
void run() {
    int *d; cudaMalloc(&d, 128 * 2 * N * 4);
    probe<MM, N><<<1, 128>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    printf("M=%d N=%d: %s\n", MM, N, cudaGetErrorString(e));
    static int h[128 * 512];
    cudaMemcpy(h, d, 128 * 2 * N * 4, cudaMemcpyDeviceToHost);
    for (int lane = 0; lane < 128; lane++) {
        int nz = 0;
        for (int c = 0; c < 2 * N; c++) nz |= h[lane * 2 * N + c] != 0;
        if (!nz) continue;
        printf("lane %3d:", lane);
        for (int c = 0; c < 2 * N; c++) {
            const int v = h[lane * 2 * N + c];
            if (v) printf(" c%d=(r%d,n%d)", c, -1, -1), printf("[%d]", v);
        }
        printf("\n");
    }
    cudaFree(d);
}

int main() {
    run<128, 16>();
    run<64, 16>();
    run<64, 24>();
    return 0;
}
