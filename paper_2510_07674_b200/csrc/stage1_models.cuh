// Fused per-particle cost + analytic gradient for the stage-1 placement models.
//
// Mapping: one thread owns one particle. Its state x (D values) and gradient g live
// in shared memory, column-major across the CTA (x[d * bs]) so every access is
// conflict-free. All loops run over scene tables with warp-uniform indices, the
// inner sphere-pair loop is fully unrolled when every body has the same sphere
// count (SPB = 1/2/4; tetrominoes are SPB=4), and per body pair the gradient is
// accumulated in registers (one +g / -g pair of updates per body pair instead of
// the reference's per-entry scatter, _interactions.py:171-177).
//
// Semantics follow the reference exactly:
//   pen = max(0, rsum - |ca - cb|); cost = sum w * pen (linear) or w * pen^2 (quadratic)
//   d cost / d ca = -w * (ca - cb) / d      (linear,    active = pen > 0 and d > 0)
//                 = -2 w pen (ca - cb) / d  (quadratic)
//   (geometry.py:131-202, _interactions.py:135-178)
#pragma once
#include "scene.cuh"

namespace spasm {

// --- one sphere pair ---------------------------------------------------------------
// Adds the UNWEIGHTED pen (or pen^2) to `cost` and returns the unweighted gradient
// scale s with d cost / d ca = -w * s * (ca - cb) (linear: s = 1/d, quadratic: s = 2 pen/d,
// 0 when inactive). Callers apply the group weight once per body pair.
//   fp32: one MUFU.RSQ per pair (d = d2 * rs, 1/d = rs). In the gradient-only path the
//   d2 clamp is dropped: d2 == 0 gives rs = inf, d = NaN, pen > 0 false -> inactive,
//   exactly the reference's "coincident centres contribute zero" rule.
template <typename R, bool WC, bool WG, bool Q>
__device__ __forceinline__ R pair_scale(R dx, R dy, R dz, R rsum, R& cost) {
  const R d2 = dx * dx + dy * dy + dz * dz;
  R d, inv;
  if constexpr (sizeof(R) == 4) {
    inv = WC ? rsqrtf(fmaxf(d2, 1e-30f)) : rsqrtf(d2);
    d = d2 * inv;
  } else {
    d = sqrt(d2);
    inv = d > R(0) ? R(1) / d : R(0);
  }
  const R pen = rsum - d;
  if constexpr (WC) {
    const R pc = pen > R(0) ? pen : R(0);
    cost += Q ? pc * pc : pc;
  }
  if constexpr (WG) {
    if constexpr (sizeof(R) == 4) return pen > R(0) ? (Q ? R(2) * pen * inv : inv) : R(0);
    else return (pen > R(0) && d2 > R(0)) ? (Q ? R(2) * pen * inv : inv) : R(0);
  }
  return R(0);
}

// weighted form (tower / generic callers): accumulates g = d cost / d ca
template <typename R, bool WC, bool WG, bool Q>
__device__ __forceinline__ void pen_pair_acc(R dx, R dy, R dz, R rsum, R w, R& cost, R& gx, R& gy, R& gz) {
  R c = R(0);
  const R s = pair_scale<R, WC, WG, Q>(dx, dy, dz, rsum, c);
  if constexpr (WC) cost += w * c;
  if constexpr (WG) {
    const R ws = -w * s;
    gx += ws * dx;
    gy += ws * dy;
    gz += ws * dz;
  }
}

// --- sphere vs static sphere ------------------------------------------------------
// fp32: cancellation-free form against huge wall spheres (R = 100 x box extent):
//   v = c - a (a = tangent point), q = |v|^2 + 2 R v.n = d^2 - R^2,
//   d - R = q / (d + R),   pen = r_c - (d - R).
// fp64: the reference's plain form rsum - |c - s| (same ops as numpy).
template <typename R, bool WC, bool WG, bool Q>
__device__ __forceinline__ void pen_static_acc(const TetrisScene<R>& sc, int st, R cx, R cy, R cz,
                                               R rc, R w, R& cost, R& gx, R& gy, R& gz) {
  if constexpr (sizeof(R) == 8) {
    pen_pair_acc<R, WC, WG, Q>(cx - sc.sx[st], cy - sc.sy[st], cz - sc.sz[st], rc + sc.sr[st], w,
                               cost, gx, gy, gz);
  } else {
    const R Rs = sc.sr[st];
    const R vx = cx - sc.ax[st], vy = cy - sc.ay[st], vz = cz - sc.az[st];
    const R q = (vx * vx + vy * vy + vz * vz) + R(2) * Rs * (vx * sc.nx[st] + vy * sc.ny[st] + vz * sc.nz[st]);
    const R d2 = Rs * Rs + q;
    const R inv = Math<R>::rsqrt_pos(d2);
    const R d = d2 * inv;
    const R pen = rc - __fdividef(q, d + Rs);
    if constexpr (WC) {
      const R pc = pen > R(0) ? pen : R(0);
      cost += Q ? w * (pc * pc) : w * pc;
    }
    if constexpr (WG) {
      const bool active = (pen > R(0)) && (d2 > R(0));
      const R f = Q ? R(2) * w * pen : w;
      const R s = active ? -f * inv : R(0);
      // diff = c - s = v + R n
      gx += s * (vx + Rs * sc.nx[st]);
      gy += s * (vy + Rs * sc.ny[st]);
      gz += s * (vz + Rs * sc.nz[st]);
    }
  }
}

// =============================================================================
// Tetris packing model (problems/tetris.py:159-245 over _interactions.py)
// =============================================================================
template <typename R, int SPB, bool FREE>
struct TetrisEval {
  using Scene = TetrisScene<R>;
  static constexpr int PER = FREE ? 4 : 3;

  // scratch: 2 * n_bodies values per thread (cos, sin of yaw)
  static __host__ __device__ int scratch_per_thread(const Scene& sc) { return FREE ? 2 * sc.n_bodies : 0; }

  template <bool WC, bool WG, bool Q>
  static __device__ __forceinline__ R run(const Scene& sc, const R* x, R* g, R* scr, int bs) {
    const int n = sc.n_bodies;
    R cost = R(0);
    if constexpr (FREE) {
      for (int b = 0; b < n; ++b) {
        R s, c;
        Math<R>::sincos_(x[(b * 4 + 3) * bs], &s, &c);
        scr[(2 * b) * bs] = c;
        scr[(2 * b + 1) * bs] = s;
      }
    }
    if constexpr (WG) {
      for (int d = 0; d < n * PER; ++d) g[d * bs] = R(0);
    }
    for (int i = 0; i < n; ++i) {
      const R pix = x[(i * PER) * bs], piy = x[(i * PER + 1) * bs], piz = x[(i * PER + 2) * bs];
      R ci = R(1), si = R(0);
      if constexpr (FREE) {
        ci = scr[(2 * i) * bs];
        si = scr[(2 * i + 1) * bs];
      }
      R gix = R(0), giy = R(0), giz = R(0), giw = R(0);
      const int a0 = sc.body_start[i];
      const int na = SPB ? SPB : sc.body_start[i + 1] - a0;

      // ---- body-body pairs (i < j), entries in C order (_interactions.py:46-60)
      for (int j = i + 1; j < n; ++j) {
        const R pjx = x[(j * PER) * bs], pjy = x[(j * PER + 1) * bs], pjz = x[(j * PER + 2) * bs];
        R cj = R(1), sj = R(0);
        if constexpr (FREE) {
          cj = scr[(2 * j) * bs];
          sj = scr[(2 * j + 1) * bs];
        }
        const int b0 = sc.body_start[j];
        const int nb = SPB ? SPB : sc.body_start[j + 1] - b0;
        R gpx = R(0), gpy = R(0), gpz = R(0), gyi = R(0), gyj = R(0), cpair = R(0);
        if constexpr (SPB > 0) {
          // preload body j's world spheres into registers
          R wbx[SPB], wby[SPB], wbz[SPB], rbx_[SPB], rby_[SPB], rb[SPB];
#pragma unroll
          for (int sb = 0; sb < SPB; ++sb) {
            const int b = b0 + sb;
            R rx = sc.lx[b], ry = sc.ly[b];
            if constexpr (FREE) {
              const R t = cj * rx - sj * ry;
              ry = sj * rx + cj * ry;
              rx = t;
            }
            rbx_[sb] = rx;
            rby_[sb] = ry;
            wbx[sb] = pjx + rx;
            wby[sb] = pjy + ry;
            wbz[sb] = pjz + sc.lz[b];
            rb[sb] = sc.rad[b];
          }
#pragma unroll
          for (int sa = 0; sa < SPB; ++sa) {
            const int a = a0 + sa;
            R rx = sc.lx[a], ry = sc.ly[a];
            if constexpr (FREE) {
              const R t = ci * rx - si * ry;
              ry = si * rx + ci * ry;
              rx = t;
            }
            const R wax = pix + rx, way = piy + ry, waz = piz + sc.lz[a];
            const R ra = sc.rad[a];
#pragma unroll
            for (int sb = 0; sb < SPB; ++sb) {
              const R dx = wax - wbx[sb], dy = way - wby[sb], dz = waz - wbz[sb];
              const R s = pair_scale<R, WC, WG, Q>(dx, dy, dz, ra + rb[sb], cpair);
              if constexpr (WG) {
                gpx += s * dx;
                gpy += s * dy;
                gpz += s * dz;
                if constexpr (FREE) {
                  gyi += s * (dy * rx - dx * ry);
                  gyj += s * (dy * rbx_[sb] - dx * rby_[sb]);
                }
              }
            }
          }
        } else {
          for (int sa = 0; sa < na; ++sa) {
            const int a = a0 + sa;
            R rx = sc.lx[a], ry = sc.ly[a];
            if constexpr (FREE) {
              const R t = ci * rx - si * ry;
              ry = si * rx + ci * ry;
              rx = t;
            }
            const R wax = pix + rx, way = piy + ry, waz = piz + sc.lz[a];
            const R ra = sc.rad[a];
            for (int sb = 0; sb < nb; ++sb) {
              const int b = b0 + sb;
              R ux = sc.lx[b], uy = sc.ly[b];
              if constexpr (FREE) {
                const R t = cj * ux - sj * uy;
                uy = sj * ux + cj * uy;
                ux = t;
              }
              const R dx = wax - (pjx + ux), dy = way - (pjy + uy), dz = waz - (pjz + sc.lz[b]);
              const R s = pair_scale<R, WC, WG, Q>(dx, dy, dz, ra + sc.rad[b], cpair);
              if constexpr (WG) {
                gpx += s * dx;
                gpy += s * dy;
                gpz += s * dz;
                if constexpr (FREE) {
                  gyi += s * (dy * rx - dx * ry);
                  gyj += s * (dy * ux - dx * uy);
                }
              }
            }
          }
        }
        if constexpr (WC) cost += sc.w_bb * cpair;
        if constexpr (WG) {
          const R wneg = -sc.w_bb;  // group weight applied once per body pair
          gpx *= wneg;
          gpy *= wneg;
          gpz *= wneg;
          gyi *= wneg;
          gyj *= wneg;
          gix += gpx;
          giy += gpy;
          giz += gpz;
          g[(j * PER) * bs] -= gpx;
          g[(j * PER + 1) * bs] -= gpy;
          g[(j * PER + 2) * bs] -= gpz;
          if constexpr (FREE) {
            giw += gyi;
            g[(j * PER + 3) * bs] -= gyj;
          }
        }
      }

      // ---- body-static pairs (walls), _interactions.py:62-73
      if (sc.n_static > 0) {
        for (int sa = 0; sa < na; ++sa) {
          const int a = a0 + sa;
          R rx = sc.lx[a], ry = sc.ly[a];
          if constexpr (FREE) {
            const R t = ci * rx - si * ry;
            ry = si * rx + ci * ry;
            rx = t;
          }
          const R wax = pix + rx, way = piy + ry, waz = piz + sc.lz[a];
          R gax = R(0), gay = R(0), gaz = R(0);
          for (int st = 0; st < sc.n_static; ++st)
            pen_static_acc<R, WC, WG, Q>(sc, st, wax, way, waz, sc.rad[a], sc.w_bs, cost, gax, gay, gaz);
          if constexpr (WG) {
            gix += gax;
            giy += gay;
            giz += gaz;
            if constexpr (FREE) giw += gay * rx - gax * ry;
          }
        }
      }

      // ---- height term (tetris.py:226-238); sign(0) == 0
      const R dz = piz - sc.z_star;
      if constexpr (WC) cost += Q ? sc.w_h * (dz * dz) : sc.w_h * fabs(dz);
      if constexpr (WG) {
        giz += Q ? sc.w_h * (R(2) * dz) : sc.w_h * (dz > R(0) ? R(1) : (dz < R(0) ? R(-1) : R(0)));
        g[(i * PER) * bs] += gix;
        g[(i * PER + 1) * bs] += giy;
        g[(i * PER + 2) * bs] += giz;
        if constexpr (FREE) g[(i * PER + 3) * bs] += giw;
      }
    }
    return cost;
  }
};

// =============================================================================
// Tower stacking model (problems/tower.py:144-322)
// =============================================================================
template <typename R, bool FREE>
struct TowerEval {
  using Scene = TowerScene<R>;
  static constexpr int PER = FREE ? 4 : 3;

  // scratch: suffix sums of (x, y) per block
  static __host__ __device__ int scratch_per_thread(const Scene& sc) { return 2 * sc.n_blocks; }

  template <bool WC, bool WG, bool Q>
  static __device__ __forceinline__ R run(const Scene& sc, const R* x, R* g, R* scr, int bs) {
    const int n = sc.n_blocks;
    R cost = R(0);
    if constexpr (WG) {
      for (int d = 0; d < n * PER; ++d) g[d * bs] = R(0);
    }
    // suffix sums from the top (tower.py:208-210: cumsum of the reversed stack)
    {
      R sxs = R(0), sys = R(0);
      for (int k = n - 1; k >= 0; --k) {
        sxs = (k == n - 1) ? x[(k * PER) * bs] : sxs + x[(k * PER) * bs];
        sys = (k == n - 1) ? x[(k * PER + 1) * bs] : sys + x[(k * PER + 1) * bs];
        scr[(2 * k) * bs] = sxs;
        scr[(2 * k + 1) * bs] = sys;
      }
    }
    // ---- stability terms, support i = 0..n-2 (tower.py:197-232, 272-292)
    R accx = R(0), accy = R(0);  // running prefix of the CoM gradient share
    for (int i = 0; i + 1 < n; ++i) {
      const R cnt = R(n - 1 - i);
      const R comx = scr[(2 * (i + 1)) * bs] / cnt, comy = scr[(2 * (i + 1) + 1) * bs] / cnt;
      const R relx = comx - x[(i * PER) * bs], rely = comy - x[(i * PER + 1) * bs];
      R lx = relx, ly = rely, c = R(1), s = R(0);
      if constexpr (FREE) {
        Math<R>::sincos_(x[(i * PER + 3) * bs], &s, &c);
        lx = c * relx + s * rely;
        ly = -s * relx + c * rely;
      }
      const R h = sc.half;
      const R clx = lx < -h ? -h : (lx > h ? h : lx);
      const R cly = ly < -h ? -h : (ly > h ? h : ly);
      const R dlx = lx - clx, dly = ly - cly;
      const R dist = Math<R>::sqrt_(dlx * dlx + dly * dly);
      if constexpr (WC) cost += Q ? sc.w_s * (dist * dist) : sc.w_s * dist;
      if constexpr (WG) {
        const R factor = sc.w_s * (Q ? R(2) * dist : (dist > R(0) ? R(1) : R(0)));
        const R ux = dist > R(0) ? dlx / dist : R(0), uy = dist > R(0) ? dly / dist : R(0);
        const R glx = factor * ux, gly = factor * uy;
        R gwx = glx, gwy = gly;
        if constexpr (FREE) {
          gwx = c * glx - s * gly;
          gwy = s * glx + c * gly;
          const R drx = -s * relx + c * rely, dry = -c * relx - s * rely;
          g[(i * PER + 3) * bs] += glx * drx + gly * dry;
        }
        accx += gwx / cnt;
        accy += gwy / cnt;
        g[((i + 1) * PER) * bs] += accx;
        g[((i + 1) * PER + 1) * bs] += accy;
        g[(i * PER) * bs] -= gwx;
        g[(i * PER + 1) * bs] -= gwy;
      }
    }
    // ---- height targets
    for (int i = 0; i < n; ++i) {
      const R dz = x[(i * PER + 2) * bs] - sc.target[i];
      if constexpr (WC) cost += Q ? sc.w_h * (dz * dz) : sc.w_h * fabs(dz);
      if constexpr (WG)
        g[(i * PER + 2) * bs] += sc.w_h * (Q ? R(2) * dz : (dz > R(0) ? R(1) : (dz < R(0) ? R(-1) : R(0))));
    }
    // ---- cube-cube pairs (rsum = side) and cube-obstacle pairs
    for (int i = 0; i < n; ++i) {
      const R pix = x[(i * PER) * bs], piy = x[(i * PER + 1) * bs], piz = x[(i * PER + 2) * bs];
      R gix = R(0), giy = R(0), giz = R(0);
      for (int j = i + 1; j < n; ++j) {
        R gx = R(0), gy = R(0), gz = R(0);
        pen_pair_acc<R, WC, WG, Q>(pix - x[(j * PER) * bs], piy - x[(j * PER + 1) * bs],
                                   piz - x[(j * PER + 2) * bs], sc.side, sc.w_c, cost, gx, gy, gz);
        if constexpr (WG) {
          gix += gx;
          giy += gy;
          giz += gz;
          g[(j * PER) * bs] -= gx;
          g[(j * PER + 1) * bs] -= gy;
          g[(j * PER + 2) * bs] -= gz;
        }
      }
      for (int o = 0; o < sc.n_obs; ++o)
        pen_pair_acc<R, WC, WG, Q>(pix - sc.ox[o], piy - sc.oy[o], piz - sc.oz[o], sc.radius + sc.orad[o],
                                   sc.w_c, cost, gix, giy, giz);
      if constexpr (WG) {
        g[(i * PER) * bs] += gix;
        g[(i * PER + 1) * bs] += giy;
        g[(i * PER + 2) * bs] += giz;
      }
    }
    return cost;
  }
};

}  // namespace spasm
