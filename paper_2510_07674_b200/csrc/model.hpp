// Host-side model object behind the opaque spasm_model handle.
#pragma once
#include <vector>

#include "../../include/spasm.h"
#include "scene.cuh"
#include "rng.cuh"

namespace spasm {

// pinned staging buffers shared by all handles (capi.cu): get a buffer of >= bytes (the size
// actually held is written to *got), put it back when the handle is done with it
cudaError_t pinned_get(void** p, size_t bytes, size_t* got);
void pinned_put(void* p, size_t bytes);
void pinned_trim();


enum class ModelKind { Tetris = 1, Tower = 2 };

// a launched, not yet collected stage-1 solve (capi.cu solve_launch / solve_collect)
struct SolvePending {
  bool active = false, graph = false;
  int dtype_size = 0, per_restart_launches = 0, rc = 0;
  spasm_solve_config cfg{};
  size_t res_bytes = 0;
  char* res_dev = nullptr;
  void* ws = nullptr;
  int64_t n_warm = 0;
  spasm_solve_report rep{};              // host-loop path: parsed result
  std::vector<double> rows, costs;
  std::vector<int64_t> idx;
};

struct Model {
  ModelKind kind;
  int dim;
  TetrisScene<float> tf;
  TetrisScene<double> td;
  TowerScene<float> wf;
  TowerScene<double> wd;
  // fp32 tile-kernel scene, valid when tile_ok (stage1_tile.cuh)
  TetrisTileScene tile;
  bool tile_ok = false;
  TowerTileScene tower_tile;  // valid when tower_tile_ok (stage1_tower_tile.cuh)
  bool tower_tile_ok = false;
  // double-precision bounds for the bit-exact sampler (numpy draws in float64)
  Bounds64 bounds;
  // pinned staging for solve results (grown on demand, never inside a kernel sequence)
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
  // cached CUDA graph of one stage-1 restart (capi.cu solve_impl) and what it was built for
  cudaGraphExec_t gexec = nullptr;
  cudaStream_t cap = nullptr;
  RestartParams* rp_dev = nullptr;
  RestartParams* rp_host = nullptr;
  struct GraphKeyPod {
    void* ws;
    void* host;
    int dtype;
    int64_t n, m;
    int k_lin, k_quad;
    double eta, alpha, eps;
    int p_return, max_restarts, sampler;
    int64_t n_warm;
    int tile;
    int tower_lanes;
  } gkey{}, gkey_seen{};
  // the solve launched by spasm_solve_launch, until spasm_solve_collect (capi.cu)
  SolvePending pend;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;

  template <typename R> const TetrisScene<R>& tetris() const;
  template <typename R> const TowerScene<R>& tower() const;
};

template <> inline const TetrisScene<float>& Model::tetris<float>() const { return tf; }
template <> inline const TetrisScene<double>& Model::tetris<double>() const { return td; }
template <> inline const TowerScene<float>& Model::tower<float>() const { return wf; }
template <> inline const TowerScene<double>& Model::tower<double>() const { return wd; }

}  // namespace spasm
