// fp32 tetris tile kernels, 8 bodies (stage1_tile.cuh).
#define SPASM_TILE_N 8
#include "stage1tile_inst.inc"
