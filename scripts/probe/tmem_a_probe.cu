// Probe: tcgen05.mma with the A operand in TMEM ([a-tmem] form) for kind::mxf4.block_scale.block32
// and kind::i8, M = 128, N = 16: (1) correctness against the host (A row r = TMEM lane r, K packed
// along 32-bit columns, element k at bits (k % 8) * 4 (fp4) / (k % 4) * 8 (i8)); (2) MMA issue
// throughput with A from shared memory vs TMEM, and tcgen05.st throughput (cycles per op per SM).
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

constexpr int N = 16;
// FP4: K = 64 per MMA (8 TMEM columns of A); I8: K = 32 per MMA (8 columns)
template <bool FP4, int KS>
__global__ void probe(const int8_t *A, const int8_t *B, int32_t *out) {
    constexpr int KM = FP4 ? 64 : 32, K = KM * KS, RB = FP4 ? K / 2 : K;   // row bytes
    __shared__ __align__(1024) uint8_t sb[N * RB];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < N * RB; i += 128) {
        const int r = i / RB, kb = i % RB;
        const int g = r / 8, j = r % 8, kc = kb / 16, x = kb % 16;
        sb[kc * (N / 8) * 128 + g * 128 + j * 16 + x] =
            FP4 ? (uint8_t)(e2m1(B[r * K + 2 * kb]) | (e2m1(B[r * K + 2 * kb + 1]) << 4)) : (uint8_t)B[r * K + kb];
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
    constexpr uint32_t ACOL = 32, SFCOL = 96;            // A at columns 32.., scales at 96..
    const uint32_t lrow = (uint32_t)(warp * 32) << 16;
    // A row tid -> TMEM lane tid, columns ACOL + 8 ks + w
    for (int ks = 0; ks < KS; ks++) {
        uint32_t w[8];
        for (int c = 0; c < 8; c++) {
            uint32_t x = 0;
            if (FP4) for (int e = 0; e < 8; e++) x |= (uint32_t)e2m1(A[tid * K + ks * 64 + 8 * c + e]) << (4 * e);
            else for (int e = 0; e < 4; e++) x |= (uint32_t)(uint8_t)A[tid * K + ks * 32 + 4 * c + e] << (8 * e);
            w[c] = x;
        }
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tmem + lrow + ACOL + 8 * ks),
                     "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]));
    }
    if (FP4) {
        const uint32_t s = 0x7f7f7f7fu;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tmem + lrow + SFCOL),
                     "r"(s), "r"(s), "r"(s), "r"(s), "r"(s), "r"(s), "r"(s), "r"(s));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
        tc_fence_after();
        for (int ks = 0; ks < KS; ks++) {
            const uint64_t bd = umma_desc(smem_u32(sb) + ks * 2 * (N / 8) * 128, (N / 8) * 128, 128);
            const uint32_t acc = ks > 0;
            if (FP4) {
                const uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(128 >> 4) << 24);
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%5], [%6], p;\n\t}\n"
                             ::"r"(tmem), "r"(tmem + ACOL + 8 * ks), "l"(bd), "r"(idesc), "r"(acc), "r"(tmem + SFCOL), "r"(tmem + SFCOL));
            } else {
                // i8: D s32 (c_format 2), a/b signed (formats 1), N, M
                const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n"
                             ::"r"(tmem), "r"(tmem + ACOL + 8 * ks), "l"(bd), "r"(idesc), "r"(acc));
            }
        }
        umma_commit(&bar);
    }
    if (tid == 0) mbar_wait(&bar, 0);
    __syncthreads();
    tc_fence_after();
    for (int c = 0; c < N; c++) {
        uint32_t v;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem + lrow + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        out[tid * N + c] = FP4 ? (int32_t)__uint_as_float(v) : (int32_t)v;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128u));
}

// Throughput: MODE 0 = fp4 MMAs with A from smem, 1 = fp4 MMAs with A from TMEM, 2 = tcgen05.st x8
// loop (all 4 warps), 3 = i8 A smem, 4 = i8 A TMEM.  ITERS ops per CTA.
template <int MODE>
__global__ void thr(int iters, unsigned long long *cyc) {
    __shared__ __align__(1024) uint8_t sa[128 * 32];
    __shared__ __align__(1024) uint8_t sb[N * 32];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 128 * 32; i += 128) sa[i] = (uint8_t)(i * 7);
    for (int i = tid; i < N * 32; i += 128) sb[i] = (uint8_t)(i * 5);
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
    const uint32_t lrow = (uint32_t)(warp * 32) << 16;
    const uint32_t s = 0x7f7f7f7fu;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tmem + lrow + 96),
                 "r"(s), "r"(s), "r"(s), "r"(s), "r"(s), "r"(s), "r"(s), "r"(s));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const unsigned long long t0 = clock64();
    if (MODE == 2) {
        for (int i = 0; i < iters; i++) {
            const uint32_t x = (uint32_t)i;
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tmem + lrow + 32 + 8 * (i & 7)),
                         "r"(x), "r"(x), "r"(x), "r"(x), "r"(x), "r"(x), "r"(x), "r"(x));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    } else if (MODE == 5 && warp > 0) {
        // concurrent TMEM stores into columns 64.. (not read by the MMAs) by warps 1-3
        for (int i = 0; i < iters; i++) {
            const uint32_t x = (uint32_t)i;
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tmem + lrow + 64 + 8 * (i & 3)),
                         "r"(x), "r"(x), "r"(x), "r"(x), "r"(x), "r"(x), "r"(x), "r"(x));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    } else if (tid == 0) {
        const uint64_t ad = umma_desc(smem_u32(sa), (128 / 8) * 128, 128);
        const uint64_t bd = umma_desc(smem_u32(sb), (N / 8) * 128, 128);
        const uint32_t idf = (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(128 >> 4) << 24);
        const uint32_t idi = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        for (int i = 0; i < iters; i++) {
            if (MODE == 0)
                asm volatile("tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%4], [%4], 1;"
                             ::"r"(tmem), "l"(ad), "l"(bd), "r"(idf), "r"(tmem + 96));
            else if (MODE >= 6)      // MODE - 4 independent accumulators, round robin
                asm volatile("tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%4], [%4], 1;"
                             ::"r"(tmem + 16 * (i % (MODE - 4))), "l"(ad), "l"(bd), "r"(idf), "r"(tmem + 96));
            else if (MODE == 1 || MODE == 5)
                asm volatile("tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%4], [%4], 1;"
                             ::"r"(tmem), "r"(tmem + 32 + 8 * (i & 7)), "l"(bd), "r"(idf), "r"(tmem + 96));
            else if (MODE == 3)
                asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 1;" ::"r"(tmem), "l"(ad), "l"(bd), "r"(idi));
            else
                asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, 1;" ::"r"(tmem), "r"(tmem + 32 + 8 * (i & 7)), "l"(bd), "r"(idi));
        }
        umma_commit(&bar);
        mbar_wait(&bar, 0);
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    if (tid == 0) cyc[blockIdx.x] = t1 - t0;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128u));
}

template <bool FP4, int KS>
void run() {
    constexpr int K = (FP4 ? 64 : 32) * KS;
    static int8_t A[128 * K], B[N * K];
    static int32_t ref[128 * N], got[128 * N];
    srand(99 + KS + FP4);
    for (int i = 0; i < 128 * K; i++) A[i] = (int8_t)(FP4 ? rand() % 9 - 4 : rand() % 256 - 128);
    for (int i = 0; i < N * K; i++) B[i] = (int8_t)(FP4 ? rand() % 9 - 4 : rand() % 256 - 128);
    for (int r = 0; r < 128; r++)
        for (int n = 0; n < N; n++) {
            int s = 0;
            for (int k = 0; k < K; k++) s += A[r * K + k] * B[n * K + k];
            ref[r * N + n] = s;
        }
    int8_t *dA, *dB; int32_t *dO;
    cudaMalloc(&dA, sizeof(A)); cudaMalloc(&dB, sizeof(B)); cudaMalloc(&dO, sizeof(got));
    cudaMemcpy(dA, A, sizeof(A), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B, sizeof(B), cudaMemcpyHostToDevice);
    cudaMemset(dO, 0, sizeof(got));
    probe<FP4, KS><<<1, 128>>>(dA, dB, dO);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(got, dO, sizeof(got), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < 128 * N; i++) bad += got[i] != ref[i];
    printf("%s A-in-TMEM K=%d: %s, mismatches %d / %d; D[0][0..2] = %d %d %d (ref %d %d %d)\n", FP4 ? "mxf4" : "i8", K,
           cudaGetErrorString(e), bad, 128 * N, got[0], got[1], got[2], ref[0], ref[1], ref[2]);
    cudaFree(dA); cudaFree(dB); cudaFree(dO);
}

template <int MODE>
void bench(int ctas_per_sm) {
    const int grid = 148 * ctas_per_sm, iters = 8192;
    unsigned long long *d, h[148 * 8];
    cudaMalloc(&d, sizeof(h));
    thr<MODE><<<grid, 128>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < grid; i++) mx = h[i] > mx ? h[i] : mx;
    const char *nm[] = {"fp4 MMA A smem", "fp4 MMA A tmem", "tcgen05.st x8 (per warp)", "i8 MMA A smem", "i8 MMA A tmem", "fp4 A tmem + 3 warps st", "fp4 A smem, 2 accumulators", "fp4 A smem, 3 accumulators", "fp4 A smem, 4 accumulators"};
    printf("%-26s ctas/SM %d: %s  %.2f cycles per op per SM\n", nm[MODE], ctas_per_sm, cudaGetErrorString(e),
           mx / ((double)iters * ctas_per_sm * (MODE == 2 ? 4 : 1)));
    cudaFree(d);
}

int main() {
    run<true, 1>();
    run<true, 2>();
    run<false, 1>();
    run<false, 3>();
    for (int c = 1; c <= 4; c *= 2) { bench<0>(c); bench<1>(c); bench<2>(c); bench<5>(c); bench<6>(c); bench<7>(c); bench<8>(c); }
    return 0;
}
