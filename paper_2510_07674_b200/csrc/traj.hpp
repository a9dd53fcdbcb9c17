// Host-side object behind the opaque spasm_traj handle: one problem's stage-2 geometry
// (reference trajopt._Geometry, trajopt.py:235-367) resident on the device in both
// precisions, plus the free-yaw placement twin (a spasm_model built by the caller).
#pragma once
#include <mutex>

#include "model.hpp"
#include "stage2.cuh"

namespace spasm {

enum TwinKind : int { kTwinNone = 0, kTwinTetris = 1, kTwinTower = 2 };

struct Traj {
  int kind = kTwinNone;           // placement twin family
  int manip = 0, B = 1, J = 0, S = 0, SB = 0, NB = 0, n_static = 0;
  TrajScene<float> hf;            // host copies
  TrajScene<double> hd;
  TrajScene<float>* df = nullptr; // device copies
  TrajScene<double>* dd = nullptr;
  const Model* twin = nullptr;    // free-yaw placement model (owned by the caller)
  void* pinned = nullptr;         // small result staging
  size_t pinned_bytes = 0;
  int64_t best_nv = -1;           // float64 values of the last accepted trajectory staged after
                                  // the result block (kAlBestOffset), -1 none (spasm_al_best_host)
  std::mutex mu;                  // guards the lazy device upload

  template <typename R> const TrajScene<R>* dev() const;
  template <typename R> const TrajScene<R>& host() const;
};

template <> inline const TrajScene<float>* Traj::dev<float>() const { return df; }
template <> inline const TrajScene<double>* Traj::dev<double>() const { return dd; }
template <> inline const TrajScene<float>& Traj::host<float>() const { return hf; }
template <> inline const TrajScene<double>& Traj::host<double>() const { return hd; }

// pinned staging layout of spasm_solve_al: the result block, then the accepted trajectory
constexpr size_t kAlBestOffset = 256;

// result block of one AL solve (device -> pinned host)
struct AlResultBlock {
  int32_t status;      // SPASM_OK / SPASM_AL_FAILURE / SPASM_LIFT_FAILURE
  int32_t kstar;       // accepted outer iteration
  int32_t best_p;      // particle index in the AL batch
  int32_t n_outers;    // outers recorded in the report (kstar + 1, or outer_iters)
  int32_t n_active;    // particles in the batch
  int32_t lift_pick_fail;  // first unreachable staged pose (-1 none)
  double objective;
  double least_violation;
  // float64 re-check of the accepted trajectory (validate, trajopt.py:1071-1153), run on the
  // device behind the AL solve: the independent check bench.solve_scene makes (bench.py:249)
  double check_violation;
  uint8_t check_feasible;
  uint8_t pad[7];
};
static_assert(sizeof(AlResultBlock) <= kAlBestOffset, "result block overlaps the staged trajectory");

}  // namespace spasm
