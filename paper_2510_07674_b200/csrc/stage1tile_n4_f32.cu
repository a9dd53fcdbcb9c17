// fp32 tetris tile kernels, 4 bodies (stage1_tile.cuh).
#define SPASM_TILE_N 4
#include "stage1tile_inst.inc"
