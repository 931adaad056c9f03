// probe_split.cu -- measurement hook for the paper's splitting multipliers (SURVEY.md 8(f) rank 2,
// P:4400-6100): ring products at p' = 383, the size of one sub-product of a one-level Karatsuba
// split of a 761-coefficient product (383 + 127 K-rows: 8 fp4 / 16 int8 K steps, N = 16 exactly
// as the sub-product's Hankel GEMM).  bench.py times 3 of these against one 761 product to turn
// DESIGN.md 8's "Karatsuba loses on the A-operand fetch" argument into a measurement.  Kinds 2 / 3:
// R/3 products at p' = 255 / 257, the sub-product sizes of the paper's 5-way R/3 multiplier
// (a 3n-coefficient product as 5 products of ~n coefficients, n = 254 for 761: H(0),
// H(1), H(-1), H(inf) of <= 254 coefficients and H(x) of 256).  Not part of the keygen path.
#include "runtime.cuh"

using namespace sntrup;
using namespace sntrup_rt;
using P383 = Params<383, 4591, 128, 1>;
using P255 = Params<255, 4591, 96, 1>;
using P257 = Params<257, 4591, 96, 1>;

template <class PQ>
static int probe_r3(uint64_t n, const void *a, const void *b, void *c, void *stream) {
    MulArgs m{};
    m.mode = MUL_ZIP;
    m.n_out = (long long)n;
    m.X = RowDesc{a, PQ::P16, 1, 1};
    m.Y = RowDesc{b, PQ::P16, 1, 1};
    m.out = c;
    m.out_stride = PQ::P16;
    m.out_bytes = 1;
    return launch_mul<PQ, 3>(m, (cudaStream_t)stream, 1, 1);
}

extern "C" int sntrup_probe_half_mul(int kind, uint64_t n, const void *a, const void *b, void *c, void *stream) {
    if (n == 0 || !a || !b || !c || kind < 0 || kind > 3) return SNTRUP_E_ARG;
    std::lock_guard<std::mutex> lk(g_mu);
    if (kind == 2) return probe_r3<P255>(n, a, b, c, stream);
    if (kind == 3) return probe_r3<P257>(n, a, b, c, stream);
    MulArgs m{};
    m.mode = MUL_ZIP;
    m.n_out = (long long)n;
    if (kind == 0) {                                      // R/3, int8 rows of P16 = 384
        m.X = RowDesc{a, P383::P16, 1, 1};
        m.Y = RowDesc{b, P383::P16, 1, 1};
        m.out = c;
        m.out_stride = P383::P16;
        m.out_bytes = 1;
        return launch_mul<P383, 3>(m, (cudaStream_t)stream, 1, 1);
    }
    m.X = RowDesc{a, P383::P8, 2, 1};                     // R/q big x big, int16 rows of P8 = 384
    m.Y = RowDesc{b, P383::P8, 2, 1};
    m.out = c;
    m.out_stride = P383::P8;
    m.out_bytes = 2;
    m.periodic = 1;
    return launch_mul<P383, 4591>(m, (cudaStream_t)stream, 2, 2);
}
