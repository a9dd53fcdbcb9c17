// fp32 ("perf") instantiation of the stage-1 kernels.
#include "stage1_launch.cuh"
#define SPASM_R float
#include "stage1_inst.inc"
