// fp32 tetris tile kernels, 5 bodies (stage1_tile.cuh).
#define SPASM_TILE_N 5
#include "stage1tile_inst.inc"
