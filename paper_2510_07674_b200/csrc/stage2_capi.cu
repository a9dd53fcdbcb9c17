// extern "C" boundary of the stage-2 (trajectory) path, declared in include/spasm.h.
//
// Replaces (reference /root/reference/pkg/src/seqplace):
//   spasm_traj_create        trajopt._build_geometry          trajopt.py:305-367
//   spasm_fk                 robot.fk_batch / yaw_jacobian_batch robot.py:160-224
//   spasm_ik_solve           robot.ik_solve_batch             robot.py:227-302
//   spasm_polish_tool_down   trajopt._polish_tool_down        trajopt.py:726-776
//   spasm_traj_evaluate      trajopt._evaluate -> trajectory_cost / al_value_and_gradient
//                                                             trajopt.py:416-723
//   spasm_traj_validate      trajopt.validate                 trajopt.py:1071-1153
//   spasm_lift               trajopt.lift_placements          trajopt.py:795-876
//   spasm_init_trajectories  trajopt.init_trajectories        trajopt.py:892-923
//   spasm_solve_al           trajopt.solve_al                 trajopt.py:936-1063
#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/spasm.h"
#include "seedseq.cuh"
#include "stage2_launch.cuh"

// launchers are instantiated in stage2_f32.cu / stage2_f64.cu only
#define SPASM_TEMPLATE_PREFIX extern
#define SPASM_R float
#include "stage2_inst.inc"
#undef SPASM_R
#define SPASM_R double
#include "stage2_inst.inc"
#undef SPASM_R
#undef SPASM_TEMPLATE_PREFIX

struct spasm_model : public spasm::Model {};
struct spasm_traj : public spasm::Traj {};

namespace spasm {

// numpy normalize_yaw on the host (geometry.py:31-38)
static double wrap_host(double a) {
  const double two_pi = 2.0 * M_PI;
  double w = std::fmod(a + M_PI, two_pi);
  if (w < 0) w += two_pi;
  w -= M_PI;
  if (w <= -M_PI) w += two_pi;
  return w;
}

template <typename R>
static void fill_scene(TrajScene<R>& s, const spasm_chain& ch, const spasm_traj_desc& d, const double* pick_pos,
                       const double* pick_yaw, const double* staged_world) {
  std::memset(&s, 0, sizeof(s));
  ChainDesc<R>& c = s.ch;
  c.J = ch.dof;
  c.S = ch.n_spheres;
  int si = 0;
  for (int j = 0; j < ch.dof; ++j) {
    c.link_start[j] = si;
    while (si < ch.n_spheres && ch.sphere_link[si] == j) ++si;
  }
  c.link_start[ch.dof] = si;
  for (int j = 0; j < ch.dof; ++j) {
    for (int k = 0; k < 3; ++k) {
      c.axis[j][k] = (R)ch.axes[3 * j + k];
      c.offset[j][k] = (R)ch.offsets[3 * j + k];
    }
    c.lo[j] = (R)ch.lower[j];
    c.hi[j] = (R)ch.upper[j];
    c.lo64[j] = ch.lower[j];
    c.hi64[j] = ch.upper[j];
    c.full_circle[j] = (ch.upper[j] - ch.lower[j]) >= 2.0 * M_PI - 1e-9;
  }
  for (int k = 0; k < 3; ++k) c.tool_t[k] = (R)ch.tool_translation[k];
  for (int k = 0; k < 9; ++k) c.tool_R[k] = (R)ch.tool_rotation[k];
  for (int q = 0; q < ch.n_spheres; ++q) {
    for (int k = 0; k < 3; ++k) c.arm_local[q][k] = (R)ch.sphere_centers[3 * q + k];
    c.arm_r[q] = (R)ch.sphere_radii[q];
  }
  s.manip = d.manipulation;
  s.B = d.manipulation ? d.n_blocks : 1;
  s.anchor = d.anchor_yaw;
  s.n_static = d.n_static;
  s.free_rows = d.rows_have_yaw;
  for (int o = 0; o < d.n_static; ++o) {
    for (int k = 0; k < 3; ++k) s.st_c[o][k] = s.st4[o][k] = (R)d.static_centers[3 * o + k];
    s.st_r[o] = s.st4[o][3] = (R)d.static_radii[o];
  }
  if (d.manipulation) {
    int q = 0;
    for (int b = 0; b < d.n_blocks; ++b) {
      s.blk_start[b] = q;
      q += d.spheres_per_block[b];
    }
    s.blk_start[d.n_blocks] = q;
    s.n_blk = q;
    for (int k = 0; k < 3; ++k) s.grasp_off[k] = (R)d.grasp_offset[k];
    s.grasp_yaw = (R)d.grasp_yaw_offset;
    for (int i = 0; i < q; ++i) {
      for (int k = 0; k < 3; ++k) {
        s.bu[i][k] = (R)(d.block_centers[3 * i + k] - d.grasp_offset[k]);
        s.staged[i][k] = s.staged4[i][k] = (R)staged_world[3 * i + k];
      }
      s.br[i] = s.staged4[i][3] = (R)d.block_radii[i];
    }
    for (int b = 0; b < d.n_blocks; ++b) {
      for (int k = 0; k < 3; ++k) {
        s.pick_pos[b][k] = (R)pick_pos[3 * b + k];
        s.pick_pos64[b][k] = pick_pos[3 * b + k];
      }
      s.pick_yaw[b] = (R)pick_yaw[b];
      s.pick_yaw64[b] = pick_yaw[b];
    }
  } else {
    for (int j = 0; j < ch.dof; ++j) {
      s.start[j] = (R)d.start[j];
      s.goal[j] = (R)d.goal[j];
    }
  }
  // fp32 fixed-obstacle lists per segment (stage2.cuh obsp): statics, then the staged spheres
  // of the later blocks, padded with far inactive dummies to whole kObsGroup-pair groups
  if constexpr (sizeof(R) == 4) {
    for (int b = 0; b < s.B; ++b) {
      const int f0 = s.manip ? s.blk_start[b + 1] : 0, f1 = s.manip ? s.n_blk : 0;
      const int n = s.n_static + (f1 - f0);
      const int np = (n + 2 * kObsGroup - 1) / (2 * kObsGroup) * kObsGroup;
      s.obs_np[b] = np;
      for (int o = 0; o < 2 * np; ++o) {
        R c[3] = {(R)1e18, (R)1e18, (R)1e18}, r = (R)0;
        if (o < s.n_static) {
          for (int k = 0; k < 3; ++k) c[k] = s.st_c[o][k];
          r = s.st_r[o];
        } else if (o < n) {
          const int q = f0 + (o - s.n_static);
          for (int k = 0; k < 3; ++k) c[k] = s.staged[q][k];
          r = s.br[q];
        }
        for (int k = 0; k < 3; ++k) s.obsp[b][o / 2][2 * k + (o & 1)] = c[k];
        s.obsp[b][o / 2][6 + (o & 1)] = r;
      }
    }
  }
}

static inline cudaStream_t as_stream2(void* s) { return reinterpret_cast<cudaStream_t>(s); }

static AlParams al_params(const spasm_al_config& c) {
  AlParams p;
  p.w_start = c.w_start;
  p.w_arm = c.w_arm;
  p.w_block = c.w_block;
  p.w_place = c.w_place;
  p.mu0 = c.mu0;
  p.beta = c.beta;
  p.lr_init = c.lr_init;
  p.lr_final = c.lr_final;
  p.eps = c.validation_epsilon;
  p.outer_iters = c.outer_iters;
  p.inner_steps = c.inner_steps;
  p.place_mode = c.place_mode;
  p.T = c.waypoints;
  return p;
}

static size_t al_up(size_t x) { return (x + 255) & ~(size_t)255; }

__global__ void k_widen(const float* __restrict__ in, int64_t n, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (double)in[i];
}

struct AlWs {
  size_t mu, lam, cons, upd, obj, viol, feas, first, nout, kstar, res, best, best64, total;
};

static AlWs al_ws_layout(const Traj& tr, int dtype, int64_t P, const spasm_al_config& c) {
  const size_t r = dtype == SPASM_F32 ? 4 : 8;
  const size_t OP = (size_t)std::max(c.outer_iters, 1) * (size_t)std::max<int64_t>(P, 1);
  AlWs L;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = al_up(off + bytes);
    return o;
  };
  L.mu = take(OP * r);
  L.lam = take(3 * OP * r);
  L.cons = take(3 * OP * r);
  L.upd = take(3 * OP * r);
  L.obj = take(OP * r);
  L.viol = take(OP * r);
  L.feas = take(OP);
  L.first = take((size_t)std::max<int64_t>(P, 1) * 4);
  L.nout = take((size_t)std::max<int64_t>(P, 1) * 4);
  L.kstar = take(16);
  L.res = take(sizeof(AlResultBlock));
  L.best = take((size_t)std::max<int64_t>(P, 1) * tr.B * c.waypoints * tr.J * r);
  L.best64 = take((size_t)tr.B * c.waypoints * tr.J * 8);  // the accepted trajectory in float64
  L.total = off;
  return L;
}

static AlRecords al_records(const AlWs& L, void* ws, const int32_t* n_active) {
  char* b = reinterpret_cast<char*>(ws);
  AlRecords rec;
  rec.mu = b + L.mu;
  rec.lam = b + L.lam;
  rec.cons = b + L.cons;
  rec.upd = b + L.upd;
  rec.obj = b + L.obj;
  rec.viol = b + L.viol;
  rec.feas = reinterpret_cast<uint8_t*>(b + L.feas);
  rec.first_feas = reinterpret_cast<int32_t*>(b + L.first);
  rec.n_outers = reinterpret_cast<int32_t*>(b + L.nout);
  rec.kstar = reinterpret_cast<int*>(b + L.kstar);
  rec.best_x = b + L.best;
  rec.n_active = n_active;
  return rec;
}

struct LiftWs {
  size_t sol, ik_ok, pol_ok, score, pen, best, okt, total;
};

static LiftWs lift_ws_layout(const Traj& tr, int dtype, int64_t P, int candidates) {
  const size_t r = dtype == SPASM_F32 ? 4 : 8;
  const size_t nt = (size_t)tr.B + (size_t)P * tr.B;
  const size_t G = nt * (size_t)std::max(1, candidates);
  LiftWs L;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = al_up(off + bytes);
    return o;
  };
  L.sol = take(G * tr.J * r);
  L.ik_ok = take(G);
  L.pol_ok = take(G);
  L.score = take(G * r);
  L.pen = take(G * r);
  L.best = take(nt * tr.J * r);
  L.okt = take(nt);
  L.total = off;
  return L;
}

// upload the scene tables + pinned result staging on first device use (creation stays
// host-only, so handles can be built and validated without a GPU)
static int ensure_device(const Traj& tc) {
  Traj& t = const_cast<Traj&>(tc);
  std::lock_guard<std::mutex> lock(t.mu);
  if (t.df && t.dd && t.pinned) return SPASM_OK;
  cudaError_t e = cudaSuccess;
  if (!t.df) e = cudaMalloc(&t.df, sizeof(TrajScene<float>));
  if (e == cudaSuccess && !t.dd) e = cudaMalloc(&t.dd, sizeof(TrajScene<double>));
  if (e == cudaSuccess) e = cudaMemcpy(t.df, &t.hf, sizeof(TrajScene<float>), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(t.dd, &t.hd, sizeof(TrajScene<double>), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !t.pinned) {
    e = pinned_get(&t.pinned, 4096, &t.pinned_bytes);
  }
  if (e != cudaSuccess) {
    set_last_error(std::string("spasm_traj device upload: ") + cudaGetErrorString(e));
    return SPASM_ERR_CUDA;
  }
  return SPASM_OK;
}

#define SPASM_TRAJ_GUARD(tr)                                        \
  do {                                                              \
    if (!(tr)) {                                                    \
      ::spasm::set_last_error("null spasm_traj handle");            \
      return SPASM_ERR_USAGE;                                       \
    }                                                               \
    const int _st = ::spasm::ensure_device(*(tr));                  \
    if (_st) return _st;                                            \
  } while (0)

#define SPASM_DTYPE_GUARD(dt)                                                       \
  do {                                                                              \
    if ((dt) != SPASM_F32 && (dt) != SPASM_F64) {                                   \
      ::spasm::set_last_error("dtype must be SPASM_F32 or SPASM_F64");              \
      return SPASM_ERR_USAGE;                                                       \
    }                                                                               \
  } while (0)

}  // namespace spasm

using namespace spasm;

extern "C" {

int spasm_traj_create(spasm_traj** out, const spasm_chain* chain, const spasm_traj_desc* desc) {
  try {
    SPASM_REQUIRE(out && chain && desc, "null argument");
    *out = nullptr;
    SPASM_REQUIRE(chain->dof >= 1 && chain->dof <= kMaxJ, "chain dof must be in [1, 8]");
    SPASM_REQUIRE(chain->n_spheres >= 0 && chain->n_spheres <= kMaxArmS, "at most 16 arm spheres");
    for (int q = 1; q < chain->n_spheres; ++q)
      SPASM_REQUIRE(chain->sphere_link[q] >= chain->sphere_link[q - 1], "arm spheres must be sorted by link");
    for (int q = 0; q < chain->n_spheres; ++q)
      SPASM_REQUIRE(chain->sphere_link[q] >= 0 && chain->sphere_link[q] < chain->dof, "sphere link out of range");
    SPASM_REQUIRE(desc->n_static >= 0 && desc->n_static <= kMaxStat2, "at most 128 static obstacle spheres");
    const bool manip = desc->manipulation != 0;
    int nb = 0, sb = 0;
    if (manip) {
      SPASM_REQUIRE(desc->n_blocks >= 1 && desc->n_blocks <= kMaxSeg, "n_blocks must be in [1, 8]");
      SPASM_REQUIRE(desc->place_model != nullptr, "manipulation problems need the free-yaw placement model");
      for (int b = 0; b < desc->n_blocks; ++b) {
        nb += desc->spheres_per_block[b];
        sb = std::max(sb, desc->spheres_per_block[b]);
      }
      SPASM_REQUIRE(nb <= kMaxBlkS, "at most 64 block spheres");
      SPASM_REQUIRE(desc->place_model->dim == 4 * desc->n_blocks, "placement twin must be free-yaw (4 per block)");
    }
    std::vector<double> pick_pos(3 * kMaxSeg, 0.0), pick_yaw(kMaxSeg, 0.0), staged((size_t)3 * std::max(nb, 1), 0.0);
    if (manip) {
      const double ox = desc->grasp_offset[0], oy = desc->grasp_offset[1], oz = desc->grasp_offset[2];
      int q = 0;
      for (int b = 0; b < desc->n_blocks; ++b) {
        const double* p = desc->staged_poses + 4 * b;
        const double yaw = wrap_host(p[3]);
        const double c = std::cos(yaw), s = std::sin(yaw);
        // grasp_pose (robot.py:325-334)
        pick_pos[3 * b] = p[0] + c * ox - s * oy;
        pick_pos[3 * b + 1] = p[1] + s * ox + c * oy;
        pick_pos[3 * b + 2] = p[2] + oz;
        pick_yaw[b] = wrap_host(yaw + desc->grasp_yaw_offset);
        // staged block spheres: local @ Rz(yaw)^T + translation (trajopt.py:346-349)
        for (int i = 0; i < desc->spheres_per_block[b]; ++i, ++q) {
          const double* l = desc->block_centers + 3 * q;
          staged[3 * q] = (l[0] * c + l[1] * (-s) + l[2] * 0.0) + p[0];
          staged[3 * q + 1] = (l[0] * s + l[1] * c + l[2] * 0.0) + p[1];
          staged[3 * q + 2] = (l[0] * 0.0 + l[1] * 0.0 + l[2] * 1.0) + p[2];
        }
      }
    }
    spasm_traj* t = new (std::nothrow) spasm_traj();
    SPASM_REQUIRE(t != nullptr, "out of host memory");
    t->manip = manip;
    t->B = manip ? desc->n_blocks : 1;
    t->J = chain->dof;
    t->S = chain->n_spheres;
    t->SB = sb;
    t->NB = nb;
    t->n_static = desc->n_static;
    t->twin = manip ? static_cast<const Model*>(desc->place_model) : nullptr;
    t->kind = !manip ? kTwinNone : (t->twin->kind == ModelKind::Tetris ? kTwinTetris : kTwinTower);
    fill_scene<float>(t->hf, *chain, *desc, pick_pos.data(), pick_yaw.data(), staged.data());
    fill_scene<double>(t->hd, *chain, *desc, pick_pos.data(), pick_yaw.data(), staged.data());
    *out = t;  // device tables are uploaded on first use (ensure_device)
    return SPASM_OK;
  } catch (...) {
    set_last_error("spasm_traj_create: unexpected host exception");
    return SPASM_ERR_USAGE;
  }
}

void spasm_traj_destroy(spasm_traj* t) {
  if (!t) return;
  if (t->df) cudaFree(t->df);
  if (t->dd) cudaFree(t->dd);
  pinned_put(t->pinned, t->pinned_bytes);
  delete t;
}

int spasm_traj_segments(const spasm_traj* t) { return t ? t->B : -1; }

int spasm_fk(const spasm_traj* t, int dtype, const void* Q, int64_t n, void* ee, void* rot, void* origins, void* axes,
             void* yaw_jacobian, void* stream) {
  SPASM_TRAJ_GUARD(t);
  SPASM_DTYPE_GUARD(dtype);
  SPASM_REQUIRE(n >= 0 && (n == 0 || (Q && ee && rot)), "bad fk arguments");
  if (dtype == SPASM_F32)
    return launch_fk<float>(*t, (const float*)Q, n, (float*)ee, (float*)rot, (float*)origins, (float*)axes,
                            (float*)yaw_jacobian, as_stream2(stream));
  return launch_fk<double>(*t, (const double*)Q, n, (double*)ee, (double*)rot, (double*)origins, (double*)axes,
                           (double*)yaw_jacobian, as_stream2(stream));
}

int spasm_ik_solve(const spasm_traj* t, int dtype, const double* target_pos, const double* target_yaw,
                   int64_t n_targets, uint64_t seed, int restarts, int max_iters, double damping, void* solutions,
                   uint8_t* success, void* errors, void* stream) {
  SPASM_TRAJ_GUARD(t);
  SPASM_DTYPE_GUARD(dtype);
  SPASM_REQUIRE(n_targets >= 0 && max_iters >= 0, "bad ik arguments");
  SPASM_REQUIRE(n_targets == 0 || (target_pos && target_yaw && solutions && success && errors), "null ik buffer");
  IkOut out;
  out.sol = solutions;
  out.ik_ok = success;
  out.pol_ok = nullptr;
  out.score = errors;
  out.pen = nullptr;
  if (dtype == SPASM_F32)
    return launch_ik<float>(*t, (int)n_targets, 1, seed, 0, restarts, max_iters, damping, target_pos, target_yaw,
                            nullptr, 0, 0, 0, out, as_stream2(stream), nullptr);
  return launch_ik<double>(*t, (int)n_targets, 1, seed, 0, restarts, max_iters, damping, target_pos, target_yaw,
                           nullptr, 0, 0, 0, out, as_stream2(stream), nullptr);
}

int spasm_polish_tool_down(const spasm_traj* t, int dtype, void* Q, const double* target_pos,
                           const double* target_yaw, int64_t n, uint8_t* ok, void* stream) {
  SPASM_TRAJ_GUARD(t);
  SPASM_DTYPE_GUARD(dtype);
  SPASM_REQUIRE(n == 0 || (Q && target_pos && target_yaw && ok), "null polish buffer");
  if (dtype == SPASM_F32)
    return launch_polish<float>(*t, (float*)Q, target_pos, target_yaw, n, ok, as_stream2(stream));
  return launch_polish<double>(*t, (double*)Q, target_pos, target_yaw, n, ok, as_stream2(stream));
}

int spasm_traj_evaluate(const spasm_traj* t, int dtype, const spasm_al_config* cfg, const void* values, int64_t P,
                        int mode, int place_mode, const void* lam, const void* mu, int want_grad, void* objective,
                        void* constraints, void* lagrangian, void* grad, void* stream) {
  SPASM_TRAJ_GUARD(t);
  SPASM_DTYPE_GUARD(dtype);
  SPASM_REQUIRE(cfg && (P == 0 || values), "null evaluate argument");
  SPASM_REQUIRE(mode == SPASM_LINEAR || mode == SPASM_QUADRATIC, "mode must be SPASM_LINEAR or SPASM_QUADRATIC");
  SPASM_REQUIRE(place_mode == SPASM_LINEAR || place_mode == SPASM_QUADRATIC, "bad place_mode");
  SPASM_REQUIRE(!want_grad || grad, "gradient buffer required");
  const AlParams prm = al_params(*cfg);
  if (dtype == SPASM_F32)
    return launch_al_eval<float>(*t, prm, (const float*)values, P, (const float*)lam, (const float*)mu, mode,
                                 place_mode, want_grad, (float*)objective, (float*)constraints, (float*)lagrangian,
                                 (float*)grad, as_stream2(stream));
  return launch_al_eval<double>(*t, prm, (const double*)values, P, (const double*)lam, (const double*)mu, mode,
                                place_mode, want_grad, (double*)objective, (double*)constraints, (double*)lagrangian,
                                (double*)grad, as_stream2(stream));
}

int spasm_traj_validate(const spasm_traj* t, int dtype, const spasm_al_config* cfg, const void* values, int64_t P,
                        uint8_t* feasible, void* violation, void* stream) {
  SPASM_TRAJ_GUARD(t);
  SPASM_DTYPE_GUARD(dtype);
  SPASM_REQUIRE(cfg && (P == 0 || (values && feasible && violation)), "null validate argument");
  const AlParams prm = al_params(*cfg);
  if (dtype == SPASM_F32)
    return launch_validate<float>(*t, prm, (const float*)values, P, feasible, (float*)violation, as_stream2(stream));
  return launch_validate<double>(*t, prm, (const double*)values, P, feasible, (double*)violation, as_stream2(stream));
}

int64_t spasm_lift_workspace_bytes(const spasm_traj* t, int dtype, int64_t P, int candidates) {
  if (!t || P < 0) return -1;
  return (int64_t)lift_ws_layout(*t, dtype, P, candidates).total;
}

int spasm_lift(const spasm_traj* t, int dtype, const double* placements, int64_t P, const int32_t* n_rows, int D,
               uint64_t seed, int candidates, void* ws, int64_t ws_bytes, void* endpoints, int32_t* kept,
               int32_t* status, void* stream) {
  SPASM_TRAJ_GUARD(t);
  SPASM_DTYPE_GUARD(dtype);
  SPASM_REQUIRE(t->manip, "point-to-point problems carry their own endpoints");
  SPASM_REQUIRE(P >= 0 && (P == 0 || placements), "bad placements");
  const int per = t->hd.free_rows ? 4 : 3;
  SPASM_REQUIRE(D == per * t->B, "placement rows have the wrong dimension");
  SPASM_REQUIRE(endpoints && kept && status && ws, "null lift buffer");
  const int cand = std::max(1, candidates);
  const LiftWs L = lift_ws_layout(*t, dtype, P, cand);
  SPASM_REQUIRE(ws_bytes >= (int64_t)L.total, "lift workspace too small");
  const int nt = t->B + (int)P * t->B;
  char* b = reinterpret_cast<char*>(ws);
  IkOut out;
  out.sol = b + L.sol;
  out.ik_ok = reinterpret_cast<uint8_t*>(b + L.ik_ok);
  out.pol_ok = reinterpret_cast<uint8_t*>(b + L.pol_ok);
  out.score = b + L.score;
  out.pen = b + L.pen;
  const int score = t->n_static > 0;
  cudaStream_t s = as_stream2(stream);
  int st;
  if (dtype == SPASM_F32) {
    st = launch_ik<float>(*t, nt, cand, seed, 1000003ull, kIkRestarts, 200, kIkDamping, nullptr, nullptr, placements,
                          D, 1, score, out, s, n_rows);
    if (st) return st;
    return launch_lift_combine<float>((const float*)out.sol, out.ik_ok, out.pol_ok, (const float*)out.pen, nt, cand,
                                      t->J, t->B, (int)P, (float*)(b + L.best), (uint8_t*)(b + L.okt), kept,
                                      (float*)endpoints, status, s, n_rows);
  }
  st = launch_ik<double>(*t, nt, cand, seed, 1000003ull, kIkRestarts, 200, kIkDamping, nullptr, nullptr, placements,
                         D, 1, score, out, s, n_rows);
  if (st) return st;
  return launch_lift_combine<double>((const double*)out.sol, out.ik_ok, out.pol_ok, (const double*)out.pen, nt, cand,
                                     t->J, t->B, (int)P, (double*)(b + L.best), (uint8_t*)(b + L.okt), kept,
                                     (double*)endpoints, status, s, n_rows);
}

int spasm_trajectory_stream_state(uint64_t seed, uint64_t out[4]) {
  if (!out) return SPASM_ERR_USAGE;
  const Pcg64State s = seedseq_pcg64_dev(seed, 1ull << 20);
  out[0] = s.state_hi;
  out[1] = s.state_lo;
  out[2] = s.inc_hi;
  out[3] = s.inc_lo;
  return SPASM_OK;
}

int spasm_init_trajectories(const spasm_traj* t, int dtype, const void* endpoints, int64_t P, int n_segments,
                            const int32_t* n_active, int k_waypoint, int k_interp, const uint64_t pcg_state[4],
                            void* out, void* stream) {
  SPASM_TRAJ_GUARD(t);
  SPASM_DTYPE_GUARD(dtype);
  SPASM_REQUIRE(k_waypoint >= 0 && k_interp >= 1, "k_waypoint >= 0 and k_interp >= 1 required");
  SPASM_REQUIRE(n_segments >= 1, "n_segments must be positive");
  SPASM_REQUIRE(P == 0 || (endpoints && out && pcg_state), "null init argument");
  Pcg64State st;
  st.state_hi = pcg_state ? pcg_state[0] : 0;
  st.state_lo = pcg_state ? pcg_state[1] : 0;
  st.inc_hi = pcg_state ? pcg_state[2] : 0;
  st.inc_lo = pcg_state ? pcg_state[3] : 1;
  if (dtype == SPASM_F32)
    return launch_init_traj<float>(*t, (const float*)endpoints, P, n_segments, n_active, k_waypoint, k_interp, st, (float*)out,
                                   as_stream2(stream));
  return launch_init_traj<double>(*t, (const double*)endpoints, P, n_segments, n_active, k_waypoint, k_interp, st, (double*)out,
                                  as_stream2(stream));
}

int64_t spasm_al_workspace_bytes(const spasm_traj* t, int dtype, int64_t P, const spasm_al_config* cfg) {
  if (!t || !cfg || P < 0) return -1;
  return (int64_t)al_ws_layout(*t, dtype, P, *cfg).total;
}

int spasm_al_records(const spasm_traj* t, int dtype, int64_t P, const spasm_al_config* cfg, void* ws,
                     void* ptrs[10]) {
  SPASM_TRAJ_GUARD(t);
  SPASM_REQUIRE(cfg && ws && ptrs, "null argument");
  const AlWs L = al_ws_layout(*t, dtype, P, *cfg);
  char* b = reinterpret_cast<char*>(ws);
  const size_t offs[10] = {L.mu, L.lam, L.cons, L.upd, L.obj, L.viol, L.feas, L.first, L.nout, L.best};
  for (int i = 0; i < 10; ++i) ptrs[i] = b + offs[i];
  return SPASM_OK;
}

int spasm_solve_al(const spasm_traj* t, int dtype, const spasm_al_config* cfg, const void* values, int64_t P,
                   const int32_t* n_active, const int32_t* lift_status, void* ws, int64_t ws_bytes, void* best_values,
                   spasm_al_result* result, void* stream) {
  SPASM_TRAJ_GUARD(t);
  SPASM_DTYPE_GUARD(dtype);
  SPASM_REQUIRE(cfg && ws && result, "null solve_al argument");
  SPASM_REQUIRE(P >= 0 && (P == 0 || values), "bad trajectory batch");
  SPASM_REQUIRE(cfg->outer_iters >= 1 && cfg->inner_steps >= 1, "outer_iters and inner_steps must be positive");
  const AlWs L = al_ws_layout(*t, dtype, P, *cfg);
  SPASM_REQUIRE(ws_bytes >= (int64_t)L.total, "AL workspace too small");
  const AlRecords rec = al_records(L, ws, n_active);
  const AlParams prm = al_params(*cfg);
  cudaStream_t s = as_stream2(stream);
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  AlResultBlock* res_dev = reinterpret_cast<AlResultBlock*>(reinterpret_cast<char*>(ws) + L.res);
  int st;
  if (dtype == SPASM_F32)
    st = launch_solve_al<float>(*t, prm, (const float*)values, P, rec, lift_status, (float*)best_values, res_dev, s);
  else
    st = launch_solve_al<double>(*t, prm, (const double*)values, P, rec, lift_status, (double*)best_values, res_dev,
                                 s);
  Traj& tm = const_cast<spasm_traj&>(*t);  // the pinned staging is the handle's internal cache
  tm.best_nv = -1;
  const int64_t nv = (int64_t)t->B * cfg->waypoints * t->J;
  if (st == SPASM_OK && best_values && tm.pinned_bytes < kAlBestOffset + (size_t)nv * 8) {
    // grow the staging so the accepted trajectory rides the one D2H below (every solve syncs
    // before it returns, so no copy still targets the old buffer)
    void* grown = nullptr;
    size_t got = 0;
    if (pinned_get(&grown, kAlBestOffset + (size_t)nv * 8, &got) != cudaSuccess) {
      st = SPASM_ERR_CUDA;
    } else {
      pinned_put(tm.pinned, tm.pinned_bytes);
      tm.pinned = grown;
      tm.pinned_bytes = got;
    }
  }
  double* best64 = nullptr;
  if (st == SPASM_OK && best_values) {
    // the float64 re-check of the accepted trajectory, queued behind the solve (its result
    // joins the one D2H copy below); on failure best_values holds no trajectory and the
    // check is ignored
    best64 = reinterpret_cast<double*>(reinterpret_cast<char*>(ws) + L.best64);
    if (dtype == SPASM_F32) {
      k_widen<<<ceil_div(nv, 256), 256, 0, s>>>((const float*)best_values, nv, best64);
      if (cudaGetLastError() != cudaSuccess) st = SPASM_ERR_CUDA;
    } else {
      if (cudaMemcpyAsync(best64, best_values, (size_t)nv * 8, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
        st = SPASM_ERR_CUDA;
    }
    if (st == SPASM_OK)
      st = launch_validate<double>(*t, prm, best64, 1, &res_dev->check_feasible, &res_dev->check_violation, s);
  }
  if (st) {
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (st == SPASM_ERR_CUDA) set_last_error("spasm_solve_al: re-check launch failed");
    return st;
  }
  cudaEventRecord(e1, s);
  AlResultBlock* host = reinterpret_cast<AlResultBlock*>(t->pinned);
  cudaError_t e = cudaMemcpyAsync(host, res_dev, sizeof(AlResultBlock), cudaMemcpyDeviceToHost, s);
  // the float64 accepted trajectory rides the same sync (spasm_al_best_host): no second
  // round trip for the caller's host copy of the result
  if (e == cudaSuccess && best64)
    e = cudaMemcpyAsync(static_cast<char*>(t->pinned) + kAlBestOffset, best64, (size_t)nv * 8, cudaMemcpyDeviceToHost,
                        s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  float ms = 0.f;
  if (e == cudaSuccess) cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (e != cudaSuccess) {
    set_last_error(std::string("spasm_solve_al: ") + cudaGetErrorString(e));
    return SPASM_ERR_CUDA;
  }
  result->status = host->status;
  result->accepted_outer = host->kstar;
  result->particle_index = host->best_p;
  result->n_outers = host->n_outers;
  result->n_particles = host->n_active;
  result->lift_pick_fail = host->lift_pick_fail;
  result->objective = host->objective;
  result->least_violation = host->least_violation;
  result->device_ms = ms;
  result->checked_violation = host->check_violation;
  result->checked_feasible = host->check_feasible;
  result->reserved = 0;
  if (best64 && host->status == SPASM_OK) tm.best_nv = nv;
  return host->status;
}

int spasm_al_best_host(const spasm_traj* t, double* out, int64_t n) {
  SPASM_REQUIRE(t != nullptr && out != nullptr, "null argument");
  SPASM_REQUIRE(t->best_nv >= 0, "no accepted trajectory staged (spasm_solve_al without best_values or not SPASM_OK)");
  SPASM_REQUIRE(n == t->best_nv, "value count mismatch");
  std::memcpy(out, static_cast<const char*>(t->pinned) + kAlBestOffset, (size_t)n * 8);
  return SPASM_OK;
}

}  // extern "C"
