// ps_761.cu -- the kernels and host orchestration of parameter set 761 (one translation unit per
// set, so the sets compile in parallel; runtime.cuh / ps_ops.cuh).
#include "ps_ops.cuh"

template struct sntrup_rt::PsOps<sntrup::P761>;
