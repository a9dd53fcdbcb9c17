// fp32 tower tile kernels (stage1_tower_tile.cuh), one instantiation per block count.
#include "stage1_launch.cuh"
#include "stage1_tower_tile.cuh"

namespace spasm {

namespace {
template <int B, int LA>
int launch_tower_la(const TowerTileScene& sc, const float* src, const uint32_t* rows, int64_t M, int k_lin,
                    int k_quad, double eta, double alpha, float* ov, float* oc, uint8_t* fl, unsigned int* fc,
                    cudaStream_t s) {
  k_schedule_tower_tile<B, LA><<<ceil_div(M * LA, 128), 128, 0, s>>>(sc, src, rows, M, k_lin, k_quad, eta, alpha, ov,
                                                                    oc, fl, fc);
  SPASM_CHECK_LAUNCH();
  return SPASM_OK;
}

template <int B>
int launch_tower(const TowerTileScene& sc, const float* src, const uint32_t* rows, int64_t M, int k_lin, int k_quad,
                 double eta, double alpha, float* ov, float* oc, uint8_t* fl, unsigned int* fc, cudaStream_t s) {
  int la = tower_lanes_option();
  if (la == 0) la = sc.n_obs <= 2 ? 1 : (sc.n_obs <= 8 ? 4 : 8);  // lanes split the cube-obstacle pairs
  switch (la) {
    case 1: return launch_tower_la<B, 1>(sc, src, rows, M, k_lin, k_quad, eta, alpha, ov, oc, fl, fc, s);
    case 2: return launch_tower_la<B, 2>(sc, src, rows, M, k_lin, k_quad, eta, alpha, ov, oc, fl, fc, s);
    case 8: return launch_tower_la<B, 8>(sc, src, rows, M, k_lin, k_quad, eta, alpha, ov, oc, fl, fc, s);
    default: return launch_tower_la<B, 4>(sc, src, rows, M, k_lin, k_quad, eta, alpha, ov, oc, fl, fc, s);
  }
}
}  // namespace

int launch_schedule_tower_tile(const Model& m, const float* src, const uint32_t* rows, int64_t M, int k_lin,
                               int k_quad, double eta, double alpha, float* ov, float* oc, uint8_t* fl,
                               unsigned int* fc, cudaStream_t s) {
  if (!m.tower_tile_ok || stage1_tile_mode() == 0 || M <= 0) return -1;
  const TowerTileScene& sc = m.tower_tile;
  switch (sc.n) {
    case 2: return launch_tower<2>(sc, src, rows, M, k_lin, k_quad, eta, alpha, ov, oc, fl, fc, s);
    case 3: return launch_tower<3>(sc, src, rows, M, k_lin, k_quad, eta, alpha, ov, oc, fl, fc, s);
    case 4: return launch_tower<4>(sc, src, rows, M, k_lin, k_quad, eta, alpha, ov, oc, fl, fc, s);
    case 5: return launch_tower<5>(sc, src, rows, M, k_lin, k_quad, eta, alpha, ov, oc, fl, fc, s);
    case 6: return launch_tower<6>(sc, src, rows, M, k_lin, k_quad, eta, alpha, ov, oc, fl, fc, s);
    case 8: return launch_tower<8>(sc, src, rows, M, k_lin, k_quad, eta, alpha, ov, oc, fl, fc, s);
    default: return -1;
  }
}

}  // namespace spasm
