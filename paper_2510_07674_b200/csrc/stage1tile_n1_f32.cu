// fp32 tetris tile kernels, 1 bodies (stage1_tile.cuh).
#define SPASM_TILE_N 1
#include "stage1tile_inst.inc"
