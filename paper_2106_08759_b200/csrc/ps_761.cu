// ps_761.cu -- the kernels and host orchestration of parameter set 761 (one translation unit per
// set, so the sets compile in parallel; runtime.cuh / ps_ops.cuh).
#include "ps_ops.cuh"

template struct sntrup_rt::PsOps<sntrup::P761>;

#if SNTRUP_JUMP_TRACE
// timing experiment: the jump-divstep decision warp's per-jump phase clocks (root 0)
extern "C" int sntrup_debug_jump_trace(long long *host, int n) {
    if (n > 128 * 8) n = 128 * 8;
    return (int)cudaMemcpyFromSymbol(host, sntrup::g_jump_trace, sizeof(long long) * n);
}
#endif
