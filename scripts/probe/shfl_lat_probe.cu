// Latency probe: dependent chains of SHFL.IDX / SHFL.DOWN, FFMA, and an STS -> __syncwarp -> LDS
// round trip, one warp, clock64 around 1024 links (the divstep decision chain's building blocks).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe(float *out, long long *cyc, float seed) {
    __shared__ float sm[64];
    const int lane = threadIdx.x;
    float x = seed + lane;
    long long t0, t1;
    // shfl idx chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; i++) x = __shfl_sync(0xffffffff, x, 1) + 1.0f;
    t1 = clock64();
    cyc[0] = t1 - t0;
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; i++) x = __shfl_down_sync(0xffffffff, x, 1) * 1.0001f;
    t1 = clock64();
    cyc[1] = t1 - t0;
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; i++) x = __fmaf_rn(x, 0.999f, 0.5f);
    t1 = clock64();
    cyc[2] = t1 - t0;
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; i++) {
        sm[lane] = x;
        __syncwarp();
        x = sm[(lane + 1) & 31] + 1.0f;
        __syncwarp();
    }
    t1 = clock64();
    cyc[3] = t1 - t0;
    // unrolled shfl chain (no loop overhead)
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < 256; i++) x = __shfl_sync(0xffffffff, x, 1) + 1.0f;
    t1 = clock64();
    cyc[4] = (t1 - t0) * 4;
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < 256; i++) x = __fmaf_rn(x, 0.999f, 0.5f);
    t1 = clock64();
    cyc[5] = (t1 - t0) * 4;
    out[lane] = x;
}

int main() {
    float *o; long long *c;
    cudaMalloc(&o, 128); cudaMallocManaged(&c, 64);
    for (int r = 0; r < 3; r++) probe<<<1, 32>>>(o, c, 1.0f);
    cudaDeviceSynchronize();
    printf("per link (cycles): shfl.idx+fadd %.1f  shfl.down+fmul %.1f  ffma %.1f  sts/syncwarp/lds+fadd %.1f  "
           "shfl.idx unrolled %.1f  ffma unrolled %.1f\n",
           c[0] / 1024.0, c[1] / 1024.0, c[2] / 1024.0, c[3] / 1024.0, c[4] / 1024.0, c[5] / 1024.0);
    return 0;
}
