// ps_1277.cu -- the kernels and host orchestration of parameter set 1277 (one translation unit per
// set, so the sets compile in parallel; runtime.cuh / ps_ops.cuh).
#include "ps_ops.cuh"

template struct sntrup_rt::PsOps<sntrup::P1277>;
