// intpeak.cuh -- integer-pipe throughput microkernels (measurement only: bench.py's roofline).
//
// BASELINE.json's metric asks for the "int-pipe % of peak"; MEASURED_PEAKS.json has no integer
// peak (SURVEY.md 8(d) "Peak definitions"), so the library measures one: each thread runs CH
// independent dependency chains of one instruction kind (inline PTX, so ptxas emits exactly that
// SASS op: IMAD, IADD3, LOP3, SHF) for ITER iterations; every block records its SM id and its
// start / end SM clock (clock64), so the host gets lane-ops per clock per SM independent of the
// clock the run happened to get.
#pragma once
#include "common.cuh"

namespace sntrup {

enum IntOp { IOP_IMAD = 0, IOP_IADD3 = 1, IOP_LOP3 = 2, IOP_SHF = 3, IOP_N = 4 };

struct IntPeakRec { unsigned long long t0, t1; unsigned smid, pad; };

template <int OP, int CH, int ITER>
__global__ void __launch_bounds__(256) int_peak_kernel(uint32_t seed, uint32_t *sink, IntPeakRec *rec) {
    uint32_t x[CH];
#pragma unroll
    for (int c = 0; c < CH; c++) x[c] = seed * (threadIdx.x + 1) + 0x9E3779B9u * c;
    const uint32_t y = seed ^ 0x5bd1e995u, z = seed + 12345u;
    __syncthreads();
    unsigned long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < ITER; it++) {
#pragma unroll
        for (int u = 0; u < 8; u++) {
#pragma unroll
            for (int c = 0; c < CH; c++) {
                if (OP == IOP_IMAD) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(y), "r"(z));
                if (OP == IOP_IADD3) asm volatile("add.u32 %0, %0, %1;" : "+r"(x[c]) : "r"(y));
                if (OP == IOP_LOP3) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(y), "r"(z));
                if (OP == IOP_SHF) asm volatile("shf.l.wrap.b32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(y), "r"(z));
            }
        }
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int c = 0; c < CH; c++) acc ^= x[c];
    if (acc == 0x12345678u) sink[threadIdx.x] = acc;      // keeps the chains alive
    if (threadIdx.x == 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        rec[blockIdx.x] = IntPeakRec{t0, t1, smid, 0};
    }
}

}  // namespace sntrup
