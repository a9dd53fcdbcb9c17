// Warp-parallel placement twin for the AL engine: the free-yaw copy of the stage-1 model
// evaluated on the placed poses (trajopt.py:281-302, 448-472, 531-539; validate's
// placement term, trajopt.py:1120-1135), spread over the 32 lanes of the AL kernel's aux
// warp instead of one thread.
//
// Work items (round-robin over lanes):
//   tetris: body pairs (i < j) with all their sphere pairs, then each body vs the statics
//           (_interactions.py:46-73, 135-178); height terms on lanes < n (tetris.py:226-238);
//   tower:  stability supports i < B-1 (tower.py:197-232, suffix CoM of the blocks above),
//           heights, cube pairs, cube-obstacle pairs (tower.py:234-322).
// Every lane accumulates its gradient contributions into its own shared-memory slot
// (4 values per body); the slots are then summed in lane order, so the result is
// deterministic (no float atomics) and identical from run to run.
#pragma once
#include "stage1_models.cuh"

namespace spasm {

// scratch (elements of R) the warp twin needs for n bodies (32 lane slot rows)
__host__ __device__ inline int twin_warp_scratch(int n) { return 2 * n + 32 * 4 * n + 4; }

template <typename R>
__device__ __forceinline__ R warp_sum_fixed(R v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

template <typename R, bool WG>
__device__ __forceinline__ void twin_reduce_slots(const R* slots, int nv, R* grad, int lane, int rows = 32) {
  if constexpr (WG) {
    __syncwarp();
    for (int k = lane; k < nv; k += 32) {
      // 4 interleaved partial sums (fixed order): the 32 loads issue back to back instead
      // of one dependent load-add chain
      R s0 = R(0), s1 = R(0), s2 = R(0), s3 = R(0);
#pragma unroll 8
      for (int l = 0; l < rows; l += 4) {
        s0 += slots[l * nv + k];
        s1 += slots[(l + 1) * nv + k];
        s2 += slots[(l + 2) * nv + k];
        s3 += slots[(l + 3) * nv + k];
      }
      grad[k] = (s0 + s1) + (s2 + s3);
    }
  }
}

// ---- tetris (free yaw; rows (x, y, z, yaw) per body) ------------------------------------
template <typename R, int SPB, bool WG, bool Q>
__device__ R twin_tetris_warp(const TetrisScene<R>& sc, const R* rows, R* grad, R* scr, int lane) {
  const int n = sc.n_bodies;
  const int nv = 4 * n;
  R* cs = scr;           // cos, sin per body
  R* gl = scr + 2 * n;   // 32 lane slots of nv values
  R* my = gl + lane * nv;
  if (lane < n) Math<R>::sincos_(rows[4 * lane + 3], &cs[2 * lane + 1], &cs[2 * lane]);
  if constexpr (WG)
    for (int k = 0; k < nv; ++k) my[k] = R(0);
  __syncwarp();
  R cost = R(0);
  const int npairs = n * (n - 1) / 2;
  const int items = npairs + (sc.n_static > 0 ? sc.body_start[n] : 0);  // + one item per sphere vs statics
  for (int it = lane; it < items; it += 32) {
    if (it < npairs) {
      int i = 0, rem = it;
      while (rem >= n - 1 - i) {
        rem -= n - 1 - i;
        ++i;
      }
      const int j = i + 1 + rem;
      const R ci = cs[2 * i], si = cs[2 * i + 1], cj = cs[2 * j], sj = cs[2 * j + 1];
      const R pix = rows[4 * i], piy = rows[4 * i + 1], piz = rows[4 * i + 2];
      const R pjx = rows[4 * j], pjy = rows[4 * j + 1], pjz = rows[4 * j + 2];
      R gpx = R(0), gpy = R(0), gpz = R(0), gyi = R(0), gyj = R(0), cpair = R(0);
      for (int a = sc.body_start[i]; a < sc.body_start[i + 1]; ++a) {
        const R rx = ci * sc.lx[a] - si * sc.ly[a], ry = si * sc.lx[a] + ci * sc.ly[a];
        const R wax = pix + rx, way = piy + ry, waz = piz + sc.lz[a];
        for (int b = sc.body_start[j]; b < sc.body_start[j + 1]; ++b) {
          const R ux = cj * sc.lx[b] - sj * sc.ly[b], uy = sj * sc.lx[b] + cj * sc.ly[b];
          const R dx = wax - (pjx + ux), dy = way - (pjy + uy), dz = waz - (pjz + sc.lz[b]);
          const R s = pair_scale<R, true, WG, Q>(dx, dy, dz, sc.rad[a] + sc.rad[b], cpair);
          if constexpr (WG) {
            gpx += s * dx;
            gpy += s * dy;
            gpz += s * dz;
            gyi += s * (dy * rx - dx * ry);
            gyj += s * (dy * ux - dx * uy);
          }
        }
      }
      cost += sc.w_bb * cpair;
      if constexpr (WG) {
        const R wneg = -sc.w_bb;
        my[4 * i] += wneg * gpx;
        my[4 * i + 1] += wneg * gpy;
        my[4 * i + 2] += wneg * gpz;
        my[4 * i + 3] += wneg * gyi;
        my[4 * j] -= wneg * gpx;
        my[4 * j + 1] -= wneg * gpy;
        my[4 * j + 2] -= wneg * gpz;
        my[4 * j + 3] -= wneg * gyj;
      }
    } else {
      const int a = it - npairs;  // movable sphere a of body i vs every static
      int i = 0;
      while (sc.body_start[i + 1] <= a) ++i;
      const R ci = cs[2 * i], si = cs[2 * i + 1];
      const R pix = rows[4 * i], piy = rows[4 * i + 1], piz = rows[4 * i + 2];
      R gx = R(0), gy = R(0), gz = R(0), gw = R(0);
      {
        const R rx = ci * sc.lx[a] - si * sc.ly[a], ry = si * sc.lx[a] + ci * sc.ly[a];
        const R wax = pix + rx, way = piy + ry, waz = piz + sc.lz[a];
        R gax = R(0), gay = R(0), gaz = R(0);
        for (int st = 0; st < sc.n_static; ++st)
          pen_static_acc<R, true, WG, Q>(sc, st, wax, way, waz, sc.rad[a], sc.w_bs, cost, gax, gay, gaz);
        if constexpr (WG) {
          gx += gax;
          gy += gay;
          gz += gaz;
          gw += gay * rx - gax * ry;
        }
      }
      if constexpr (WG) {
        my[4 * i] += gx;
        my[4 * i + 1] += gy;
        my[4 * i + 2] += gz;
        my[4 * i + 3] += gw;
      }
    }
  }
  if (lane < n) {  // height term, sign(0) == 0
    const R dz = rows[4 * lane + 2] - sc.z_star;
    cost += Q ? sc.w_h * (dz * dz) : sc.w_h * fabs(dz);
    if constexpr (WG) my[4 * lane + 2] += Q ? sc.w_h * (R(2) * dz) : sc.w_h * (dz > R(0) ? R(1) : (dz < R(0) ? R(-1) : R(0)));
  }
  cost = warp_sum_fixed(cost);
  twin_reduce_slots<R, WG>(gl, nv, grad, lane);
  __syncwarp();
  return cost;
}

// ---- tower (free yaw; rows (x, y, z, yaw) per block) ------------------------------------
// cube-obstacle pairs: G lanes per cube, lane l owns cube l / G and obstacles
// o = l % G, l % G + G, ... (register accumulation, one slot update per lane)
template <typename R, bool WG, bool Q>
__device__ __forceinline__ void twin_tower_obstacles(const TowerScene<R>& sc, const R* rows, R* my, int lane,
                                                     R& cost) {
  const int n = sc.n_blocks;
  const int G = 32 / n;
  if (lane < n * G) {
    const int i = lane / G;
    const R cx = rows[4 * i], cy = rows[4 * i + 1], cz = rows[4 * i + 2];
    R gx = R(0), gy = R(0), gz = R(0);
    for (int o = lane - i * G; o < sc.n_obs; o += G)
      pen_pair_acc<R, true, WG, Q>(cx - sc.ox[o], cy - sc.oy[o], cz - sc.oz[o], sc.radius + sc.orad[o], sc.w_c,
                                   cost, gx, gy, gz);
    if constexpr (WG) {
      R* mi = my + 4 * i;
      const R a0 = mi[0], a1 = mi[1], a2 = mi[2];
      mi[0] = a0 + gx;
      mi[1] = a1 + gy;
      mi[2] = a2 + gz;
    }
  }
}

// Items [it_lo, it_hi) of the tower twin (supports i < B-1, heights, cube pairs) and, when
// `obstacles`, the cube-obstacle pairs, accumulated into this lane's slot row `my` (zeroed
// here); returns the lane's cost.
template <typename R, bool WG, bool Q>
__device__ R twin_tower_core(const TowerScene<R>& sc, const R* rows, R* my, int lane, int it_lo, int it_hi,
                             bool obstacles) {
  const int n = sc.n_blocks;
  const int nv = 4 * n;
  if constexpr (WG)
    for (int k = 0; k < nv; ++k) my[k] = R(0);
  R cost = R(0);
  const int n_stab = n - 1, n_pair = n * (n - 1) / 2;
  const int items = n_stab + n + n_pair;  // the cube-obstacle pairs follow separately
  for (int it = it_lo + lane; it < (it_hi < items ? it_hi : items); it += 32) {
    if (it < n_stab) {  // support i: suffix CoM of the blocks above, in i's yaw frame
      const int i = it;
      R sxs = R(0), sys = R(0);
      for (int k = n - 1; k > i; --k) {
        sxs = (k == n - 1) ? rows[4 * k] : sxs + rows[4 * k];
        sys = (k == n - 1) ? rows[4 * k + 1] : sys + rows[4 * k + 1];
      }
      const R cnt = R(n - 1 - i);
      const R comx = sxs / cnt, comy = sys / cnt;
      const R relx = comx - rows[4 * i], rely = comy - rows[4 * i + 1];
      R s, c;
      Math<R>::sincos_(rows[4 * i + 3], &s, &c);
      const R lx = c * relx + s * rely, ly = -s * relx + c * rely;
      const R h = sc.half;
      const R clx = lx < -h ? -h : (lx > h ? h : lx);
      const R cly = ly < -h ? -h : (ly > h ? h : ly);
      const R dlx = lx - clx, dly = ly - cly;
      const R dist = Math<R>::sqrt_(dlx * dlx + dly * dly);
      cost += Q ? sc.w_s * (dist * dist) : sc.w_s * dist;
      if constexpr (WG) {
        const R factor = sc.w_s * (Q ? R(2) * dist : (dist > R(0) ? R(1) : R(0)));
        const R ux = dist > R(0) ? dlx / dist : R(0), uy = dist > R(0) ? dly / dist : R(0);
        const R glx = factor * ux, gly = factor * uy;
        const R gwx = c * glx - s * gly, gwy = s * glx + c * gly;
        const R drx = -s * relx + c * rely, dry = -c * relx - s * rely;
        // slot updates as load-all / store-all (distinct slots; the shared-memory RMWs
        // otherwise serialise on possible aliasing)
        R* mi = my + 4 * i;
        const R m0 = mi[0], m1 = mi[1], m3 = mi[3];
        mi[3] = m3 + (glx * drx + gly * dry);
        mi[0] = m0 - gwx;
        mi[1] = m1 - gwy;
        const R ax = gwx / cnt, ay = gwy / cnt;
        for (int k = i + 1; k < n; ++k) {
          const R mx = my[4 * k], myy = my[4 * k + 1];
          my[4 * k] = mx + ax;
          my[4 * k + 1] = myy + ay;
        }
      }
    } else if (it < n_stab + n) {  // height target (i+1) * side
      const int i = it - n_stab;
      const R dz = rows[4 * i + 2] - sc.target[i];
      cost += Q ? sc.w_h * (dz * dz) : sc.w_h * fabs(dz);
      if constexpr (WG) my[4 * i + 2] += sc.w_h * (Q ? R(2) * dz : (dz > R(0) ? R(1) : (dz < R(0) ? R(-1) : R(0))));
    } else if (it < n_stab + n + n_pair) {  // cube pair (rsum = side)
      int i = 0, rem = it - n_stab - n;
      while (rem >= n - 1 - i) {
        rem -= n - 1 - i;
        ++i;
      }
      const int j = i + 1 + rem;
      R gx = R(0), gy = R(0), gz = R(0);
      pen_pair_acc<R, true, WG, Q>(rows[4 * i] - rows[4 * j], rows[4 * i + 1] - rows[4 * j + 1],
                                   rows[4 * i + 2] - rows[4 * j + 2], sc.side, sc.w_c, cost, gx, gy, gz);
      if constexpr (WG) {
        R* mi = my + 4 * i;
        R* mj = my + 4 * j;
        const R a0 = mi[0], a1 = mi[1], a2 = mi[2], b0 = mj[0], b1 = mj[1], b2 = mj[2];
        mi[0] = a0 + gx;
        mi[1] = a1 + gy;
        mi[2] = a2 + gz;
        mj[0] = b0 - gx;
        mj[1] = b1 - gy;
        mj[2] = b2 - gz;
      }
    }
  }
  if (obstacles) twin_tower_obstacles<R, WG, Q>(sc, rows, my, lane, cost);
  return cost;
}

// The whole tower twin on the aux warp (the tile warps are the longer path through the
// step: handing its parts to them lengthened the step).
template <typename R, bool WG, bool Q>
__device__ R twin_tower_warp(const TowerScene<R>& sc, const R* rows, R* grad, R* scr, int lane) {
  const int n = sc.n_blocks;
  const int nv = 4 * n;
  R* gl = scr + 2 * n;
  R cost = twin_tower_core<R, WG, Q>(sc, rows, gl + lane * nv, lane, 0, 1 << 30, true);
  cost = warp_sum_fixed(cost);
  twin_reduce_slots<R, WG>(gl, nv, grad, lane, 32);
  __syncwarp();
  return cost;
}

// Cost of the placement twin on all 32 lanes of the calling warp; grad (4 per body)
// written when want_grad.
template <typename R, int KIND, int SPB, class TS>
__device__ R twin_warp(const TS& ts, const R* rows, R* grad, R* scr, int lane, bool want_grad, bool quad) {
  if constexpr (KIND == 1) {
    if (want_grad)
      return quad ? twin_tetris_warp<R, SPB, true, true>(ts, rows, grad, scr, lane)
                  : twin_tetris_warp<R, SPB, true, false>(ts, rows, grad, scr, lane);
    return quad ? twin_tetris_warp<R, SPB, false, true>(ts, rows, grad, scr, lane)
                : twin_tetris_warp<R, SPB, false, false>(ts, rows, grad, scr, lane);
  } else if constexpr (KIND == 2) {
    if (want_grad)
      return quad ? twin_tower_warp<R, true, true>(ts, rows, grad, scr, lane)
                  : twin_tower_warp<R, true, false>(ts, rows, grad, scr, lane);
    return quad ? twin_tower_warp<R, false, true>(ts, rows, grad, scr, lane)
                : twin_tower_warp<R, false, false>(ts, rows, grad, scr, lane);
  } else {
    return R(0);
  }
}

}  // namespace spasm
