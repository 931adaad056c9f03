// Probe: "transposed" Hankel GEMM for one convolution on tcgen05.mma kind::i8 with M = 64.
//   c[16 m + n] = sum_j a[j] b[16 m + n - j]
// M side (A descriptor): row m' = 63 - m is the window Zr[16 m' + k] of the reversed b
// (Zr[x] = b[1023 - x]) -- a plain VIEW of one byte array with LBO = 16 B (K chunks 16 B apart,
// overlapping the next row), SBO = 128 B; K step s at +32 B.  No materialised operand.
// N side (B descriptor): row n = 0..N-1 is the sliding window of a (16-byte row rho = hA[rho..rho+15],
// hA[x] = a[x - 15]), LBO = 256 B, SBO = 128 B; K step s at +512 B.
// Question: does the descriptor hardware accept LBO = 16 (a K chunk that overlaps the next rows)?
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../../paper_2106_08759_b200/csrc/tcmul.cuh"
using namespace sntrup;

constexpr int P = 500, KS = (P + 15 + 31) / 32, K = 32 * KS;
constexpr int ZLEN = 16 * 64 + K + 64;          // Zr bytes read by rows 0..63 over all K steps
constexpr int WROWS = K + 32;                    // window rows

template <int N>
__global__ void probe(const int8_t *a, const int8_t *b, int *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *W = sm;                              // WROWS x 16 B
    uint8_t *Z = sm + (WROWS * 16 + 127) / 128 * 128;
    uint64_t *bar = reinterpret_cast<uint64_t *>(Z + (ZLEN + 127) / 128 * 128);
    uint32_t *slot = reinterpret_cast<uint32_t *>(bar + 1);
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < WROWS * 16; i += 128) {
        const int rho = i / 16, kk = i % 16, j = rho + kk - 15;
        W[i] = (j >= 0 && j < P) ? (uint8_t)a[j] : 0;
    }
    for (int x = tid; x < ZLEN; x += 128) {
        const int j = 1023 - x;
        Z[x] = (j >= 0 && j < P) ? (uint8_t)b[j] : 0;
    }
    if (tid == 0) { mbar_init(bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(64u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    if (warp == 0) {
        const uint32_t idesc = umma_idesc_i8(N, 64);
        const uint64_t ad0 = umma_desc(smem_u32(Z), 16, 128);
        const uint64_t bd0 = umma_desc(smem_u32(W), 256, 128);
        for (int ks = 0; ks < KS; ks++)
            umma_i8_w(tmem, ad0 + (uint64_t)((ks * 32) >> 4), bd0 + (uint64_t)((ks * 512) >> 4), idesc, ks > 0 ? 1u : 0u);
        umma_commit_w(bar);
    }
    if (tid == 0) mbar_wait(bar, 0);
    __syncthreads();
    tc_fence_after();
    const uint32_t la = tmem + ((uint32_t)(warp * 32) << 16);
    int v[16];
    for (int c = 0; c < N; c += 16) {
        tmem_ld16(la + c, v);
        tmem_ld_wait();
        for (int i = 0; i < 16; i++) out[tid * N + c + i] = v[i];
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64u));
}

template <int N>
int run() {
    static int8_t ha[P], hb[P];
    srand(7 + N);
    for (int i = 0; i < P; i++) { ha[i] = (int8_t)(rand() % 61 - 30); hb[i] = (int8_t)(rand() % 61 - 30); }
    int8_t *da, *db; int *dout;
    cudaMalloc(&da, P); cudaMalloc(&db, P); cudaMalloc(&dout, 128 * N * 4);
    cudaMemcpy(da, ha, P, cudaMemcpyHostToDevice); cudaMemcpy(db, hb, P, cudaMemcpyHostToDevice);
    const int smem = (WROWS * 16 + 127) / 128 * 128 + (ZLEN + 127) / 128 * 128 + 64;
    cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    probe<N><<<1, 128, smem>>>(da, db, dout);
    cudaError_t e = cudaDeviceSynchronize();
    printf("N=%d: %s\n", N, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    static int h[128 * 64];
    cudaMemcpy(h, dout, 128 * N * 4, cudaMemcpyDeviceToHost);
    // expected: thread (warp w, lane l < 16) = row m' = 16 w + l, block m = 63 - m';
    // column n < 16: c[16 m + n]; columns 16..N-1 (second window group = rows 16.. of the same
    // sliding window, i.e. a shifted by 16 more): c[16 m + n]
    long bad = 0, checked = 0;
    for (int w = 0; w < 4; w++)
        for (int l = 0; l < 16; l++) {
            const int mp = 16 * w + l, m = 63 - mp;
            for (int n = 0; n < N; n++) {
                const int i = 16 * m + n;
                long c = 0;
                for (int j = 0; j < P; j++) { const int t = i - j; if (t >= 0 && t < P) c += (long)ha[j] * hb[t]; }
                const int got = h[(32 * w + l) * N + n];
                checked++;
                if (got != (int)c) { if (bad < 8) printf("  mismatch row %d col %d: got %d want %ld\n", mp, n, got, c); bad++; }
            }
        }
    printf("N=%d: %ld of %ld mismatches\n", N, bad, checked);
    cudaFree(da); cudaFree(db); cudaFree(dout);
    return bad != 0;
}

int main() {
    int rc = run<16>();
    rc |= run<32>();
    return rc;
}
