// fp64 ("parity") instantiation of the stage-2 kernels; built with -fmad=false so each
// operation rounds like the reference's numpy float64 expression.
#include "stage2_launch.cuh"
#define SPASM_R double
#include "stage2_inst.inc"
