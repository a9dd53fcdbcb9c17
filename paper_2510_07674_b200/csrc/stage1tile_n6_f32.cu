// fp32 tetris tile kernels, 6 bodies (stage1_tile.cuh).
#define SPASM_TILE_N 6
#include "stage1tile_inst.inc"
