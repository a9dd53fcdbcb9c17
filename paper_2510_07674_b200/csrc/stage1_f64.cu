// fp64 ("parity") instantiation of the stage-1 kernels. Built with -fmad=false so each
// multiply/add rounds separately, as numpy's float64 ufuncs do.
#include "stage1_launch.cuh"
#define SPASM_R double
#include "stage1_inst.inc"
