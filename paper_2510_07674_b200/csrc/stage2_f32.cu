// fp32 ("perf") instantiation of the stage-2 kernels.
#include "stage2_launch.cuh"
#define SPASM_R float
#include "stage2_inst.inc"
