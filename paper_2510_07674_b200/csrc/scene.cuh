// Device-resident scene tables for the stage-1 placement cost models.
//
// These are POD structs passed BY VALUE as kernel parameters: every table read in
// the pair loops is warp-uniform, so it is served from the constant bank (LDC /
// direct c[0x0][..] operands) with no shared-memory traffic and no divergence.
//
//   TetrisScene  <- SphereInteractions tables + TetrisCostModel terms
//                   (reference problems/_interactions.py:23-93, problems/tetris.py:159-245)
//   TowerScene   <- TowerCostModel terms (reference problems/tower.py:144-322)
#pragma once
#include "common.cuh"

namespace spasm {

constexpr int kMaxBodies = 16;    // movable bodies (blocks) per tetris scene
constexpr int kMaxMov = 128;      // movable spheres in total
constexpr int kMaxStatic = 32;    // static spheres (walls)
constexpr int kMaxDim = 128;      // particle state dimension D
constexpr int kMaxTowerBlocks = 32;
constexpr int kMaxObstacles = 64;

// float64 clamp/sampling bounds (numpy draws and clamps warm seeds in float64)
struct Bounds64 {
  double lo[kMaxDim];
  double hi[kMaxDim];
};

template <typename R>
struct TetrisScene {
  int n_bodies;                     // n
  int n_mov;                        // S_mov
  int n_static;                     // walls
  int free_yaw;                     // row layout (x,y,z,yaw) per block if 1 else (x,y,z)
  int dim;                          // n * (3 + free_yaw)
  int spb;                          // spheres per body if uniform, else 0
  int body_start[kMaxBodies + 1];   // sphere index range per body (C order, tetris.py:203-210)
  R lx[kMaxMov], ly[kMaxMov], lz[kMaxMov], rad[kMaxMov];  // body-local centres, radii
  // static spheres: centre + radius (fp64 path, identical to numpy's form) and the
  // cancellation-free anchor form used by the fp32 path: tangent point a = s + R n
  // and unit normal n, so |c-s|^2 - R^2 = |v|^2 + 2R v.n with v = c - a small.
  R sx[kMaxStatic], sy[kMaxStatic], sz[kMaxStatic], sr[kMaxStatic];
  R ax[kMaxStatic], ay[kMaxStatic], az[kMaxStatic];
  R nx[kMaxStatic], ny[kMaxStatic], nz[kMaxStatic];
  R w_bb, w_bs, w_h, z_star;        // PackingWeights + packing plane
  R lower[kMaxDim], upper[kMaxDim]; // clamp box (tetris.py:174-187)
};

template <typename R>
struct TowerScene {
  int n_blocks;                     // B (>= 2)
  int n_obs;                        // O
  int free_yaw;
  int dim;
  R side, half, radius;             // cube edge, footprint half-width, inscribed sphere radius
  R target[kMaxTowerBlocks];        // (i+1)*side (tower.py:100-102)
  R ox[kMaxObstacles], oy[kMaxObstacles], oz[kMaxObstacles], orad[kMaxObstacles];
  R w_s, w_h, w_c;                  // TowerWeights
  R lower[kMaxDim], upper[kMaxDim];
};

// fp32 tile-kernel scene (stage1_tile.cuh): the tetris scenes with 4 spheres per body of
// one radius, 4 wall spheres, fixed yaw and at most 8 bodies.
constexpr int kTileMaxBodies = 8;
constexpr int kTileSpb = 4;
constexpr int kTileWalls = 4;

// Host-built compact scene for the tile kernel (scalar + duplicated-pair copies of every
// constant the pair loops read, so packed ops take them as uniform-register operands).
struct TetrisTileScene {
  int n;
  float lx[kTileMaxBodies * kTileSpb], ly[kTileMaxBodies * kTileSpb], lz[kTileMaxBodies * kTileSpb];
  // the same offsets as packed pairs (spheres 2k, 2k+1 of the table) for f32x2 operands
  unsigned long long px[kTileMaxBodies * kTileSpb / 2], py[kTileMaxBodies * kTileSpb / 2],
      pz[kTileMaxBodies * kTileSpb / 2];
  // walls in box_wall_spheres order (+x, -x, +y, -y inward normals): tangent-point
  // coordinate along each wall's axis, the shared off-axis tangent coordinates, radius R
  float wall_a[kTileWalls], wall_ay_x, wall_ax_y, wall_az;
  float wr, wr2, two_wr;
  // packed wall constants (x walls, y walls as f32x2 pairs): tangent coordinates (a0, a1),
  // (a2, a3); (2R, -2R); (R, -R); and duplicated R^2, R, r
  unsigned long long wa_x, wa_y, two_wr_pm, wr_pm, wr2_d, wr_d, r_d;
  unsigned long long rs_d, m1_d, tiny_d, k_bs_d;  // duplicated rsum, -1, 1e-30, -2 w_bs
  float r, rs, rs2;  // uniform sphere radius, rsum = 2r, rsum^2
  float w_bb, w_bs, w_h, z_star;
  float lower[kTileMaxBodies * 3], upper[kTileMaxBodies * 3];
};

// fp32 tile-kernel scene for the tower scenes (stage1_tower_tile.cuh): fixed yaw, at most
// kTowerTileMaxBlocks cubes, obstacles split over the lanes from a shared-memory copy.
constexpr int kTowerTileMaxBlocks = 8;
struct TowerTileScene {
  int n, n_obs;
  float side, half, radius;
  float target[kTowerTileMaxBlocks];
  float ox[kMaxObstacles], oy[kMaxObstacles], oz[kMaxObstacles], orad[kMaxObstacles];
  float w_s, w_h, w_c;
  float lower[kTowerTileMaxBlocks * 3], upper[kTowerTileMaxBlocks * 3];
};

// Perf-mode particle update (north_star item 4; not in the reference). The default
// (adam = 0, noise = 0) is the reference's clamped gradient step (particle_opt.py:214-228)
// and every parity path uses it. adam: Adam moments with bias correction, scaled by the
// reference's learning-rate schedule. noise: Gaussian perturbation with std
// noise * (upper - lower) per dimension, annealed linearly to 0 over the linear phase,
// drawn from Philox4x32-10 keyed by (seed, restart, particle, step).
struct StepRule {
  int adam;
  float b1, b2, eps;
  float noise;
  uint64_t seed;
  uint32_t restart;
  __host__ __device__ bool is_reference() const { return adam == 0 && noise == 0.f; }
};

}  // namespace spasm
