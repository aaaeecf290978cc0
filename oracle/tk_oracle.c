/*
 * tk_oracle.c -- CPU ORACLE (test infrastructure only; never the product path).
 *
 * A plain-C, float64 restatement of the reference projector kernels in
 * /root/reference/pkg/src/tomokit/_kernels.py.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this library, and
 * only as the checker or the timed CPU baseline.
 *
 * Every function mirrors one numba kernel statement for statement: same loop
 * order per output element, same float64 operation order, no FMA contraction
 * (built with -ffp-contract=off), so outputs are bit-identical to the numba
 * reference (pinned by tests/test_oracle_golden.py against fixtures produced
 * by importing the reference itself, tests/golden/make_golden.py).
 *
 * Parallelism is over output elements (OpenMP), exactly like numba prange:
 * each output is written by one iteration in a fixed order, so results do not
 * depend on the thread count (reference _kernels.py:1-7).
 *
 * The *_transpose functions are NOT in the reference: they are the exact
 * matrix transposes of the ray-driven forward operators (the reference only
 * materialises A densely, projectors.py:294-324).  They serve as the oracle
 * for the matched-adjoint kernels.  They run serially (scatter).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define TINY 1e-12

static inline double dmax(double a, double b) { return a > b ? a : b; }
static inline double dmin(double a, double b) { return a < b ? a : b; }

/* _kernels.py:27-49 (_clip_ray_2d).  Returns 0 and sets t0 >= t1 when empty. */
static void clip_ray_2d(double px, double py, double dx, double dy, double hx,
                        double hy, double *t0o, double *t1o) {
  double t0 = -1e300, t1 = 1e300;
  if (fabs(dx) > TINY) {
    double ta = (-hx - px) / dx, tb = (hx - px) / dx;
    t0 = dmax(t0, dmin(ta, tb));
    t1 = dmin(t1, dmax(ta, tb));
  } else if (px < -hx || px > hx) {
    *t0o = 1.0; *t1o = 0.0; return;
  }
  if (fabs(dy) > TINY) {
    double ta = (-hy - py) / dy, tb = (hy - py) / dy;
    t0 = dmax(t0, dmin(ta, tb));
    t1 = dmin(t1, dmax(ta, tb));
  } else if (py < -hy || py > hy) {
    *t0o = 1.0; *t1o = 0.0; return;
  }
  *t0o = t0; *t1o = t1;
}

/* _kernels.py:52-77 (_clip_ray_3d). */
static void clip_ray_3d(double px, double py, double pz, double dx, double dy,
                        double dz, double hx, double hy, double hz, double *t0o,
                        double *t1o) {
  double t0 = -1e300, t1 = 1e300;
  if (fabs(dx) > TINY) {
    double ta = (-hx - px) / dx, tb = (hx - px) / dx;
    t0 = dmax(t0, dmin(ta, tb));
    t1 = dmin(t1, dmax(ta, tb));
  } else if (px < -hx || px > hx) {
    *t0o = 1.0; *t1o = 0.0; return;
  }
  if (fabs(dy) > TINY) {
    double ta = (-hy - py) / dy, tb = (hy - py) / dy;
    t0 = dmax(t0, dmin(ta, tb));
    t1 = dmin(t1, dmax(ta, tb));
  } else if (py < -hy || py > hy) {
    *t0o = 1.0; *t1o = 0.0; return;
  }
  if (fabs(dz) > TINY) {
    double ta = (-hz - pz) / dz, tb = (hz - pz) / dz;
    t0 = dmax(t0, dmin(ta, tb));
    t1 = dmin(t1, dmax(ta, tb));
  } else if (pz < -hz || pz > hz) {
    *t0o = 1.0; *t1o = 0.0; return;
  }
  *t0o = t0; *t1o = t1;
}

/*
 * _kernels.py:80-114 (_march_2d).  volp is the (ny+2, nx+2) zero-padded volume.
 * When `adj` is non-NULL the function instead scatters `yval` times the same
 * interpolation weights into adj (the exact transpose), returning 0.
 */
static double march_2d(const double *volp, int nyp, int nxp, double sy,
                       double sx, double px, double py, double dx, double dy,
                       double step, double *adj, double yval) {
  int ny = nyp - 2, nx = nxp - 2;
  double cy = (ny - 1) / 2.0 + 1.0;
  double cx = (nx - 1) / 2.0 + 1.0;
  double t0, t1;
  clip_ray_2d(px, py, dx, dy, (nx + 1) * sx / 2.0, (ny + 1) * sy / 2.0, &t0, &t1);
  if (t0 >= t1) return 0.0;
  double acc = 0.0;
  double t = t0;
  while (t < t1 - TINY) {
    double seg = step;
    if (t + seg > t1) seg = t1 - t;
    double tm = t + 0.5 * seg;
    double fx = (px + tm * dx) / sx + cx;
    double fy = (py + tm * dy) / sy + cy;
    long ix = (long)floor(fx);
    long iy = (long)floor(fy);
    if (0 <= ix && ix < nx + 1 && 0 <= iy && iy < ny + 1) {
      double wx = fx - ix;
      double wy = fy - iy;
      if (adj) {
        double g = yval * seg;
        adj[iy * nxp + ix] += g * ((1.0 - wx) * (1.0 - wy));
        adj[iy * nxp + ix + 1] += g * (wx * (1.0 - wy));
        adj[(iy + 1) * nxp + ix] += g * ((1.0 - wx) * wy);
        adj[(iy + 1) * nxp + ix + 1] += g * (wx * wy);
      } else {
        double val = volp[iy * nxp + ix] * (1.0 - wx) * (1.0 - wy) +
                     volp[iy * nxp + ix + 1] * wx * (1.0 - wy) +
                     volp[(iy + 1) * nxp + ix] * (1.0 - wx) * wy +
                     volp[(iy + 1) * nxp + ix + 1] * wx * wy;
        acc += val * seg;
      }
    }
    t += seg;
  }
  return acc;
}

/* _kernels.py:117-157 (_march_3d); same transpose convention as march_2d. */
static double march_3d(const double *volp, int nzp, int nyp, int nxp, double sz,
                       double sy, double sx, double px, double py, double pz,
                       double dx, double dy, double dz, double step, double *adj,
                       double yval) {
  int nz = nzp - 2, ny = nyp - 2, nx = nxp - 2;
  double cz = (nz - 1) / 2.0 + 1.0;
  double cy = (ny - 1) / 2.0 + 1.0;
  double cx = (nx - 1) / 2.0 + 1.0;
  double t0, t1;
  clip_ray_3d(px, py, pz, dx, dy, dz, (nx + 1) * sx / 2.0, (ny + 1) * sy / 2.0,
              (nz + 1) * sz / 2.0, &t0, &t1);
  if (t0 >= t1) return 0.0;
  const long sxy = (long)nyp * nxp;
  double acc = 0.0;
  double t = t0;
  while (t < t1 - TINY) {
    double seg = step;
    if (t + seg > t1) seg = t1 - t;
    double tm = t + 0.5 * seg;
    double fx = (px + tm * dx) / sx + cx;
    double fy = (py + tm * dy) / sy + cy;
    double fz = (pz + tm * dz) / sz + cz;
    long ix = (long)floor(fx);
    long iy = (long)floor(fy);
    long iz = (long)floor(fz);
    if (0 <= ix && ix < nx + 1 && 0 <= iy && iy < ny + 1 && 0 <= iz && iz < nz + 1) {
      double wx = fx - ix;
      double wy = fy - iy;
      double wz = fz - iz;
      long b = iz * sxy + iy * nxp + ix;
      if (adj) {
        double g = yval * seg;
        adj[b] += g * ((1.0 - wx) * (1.0 - wy) * (1.0 - wz));
        adj[b + 1] += g * (wx * (1.0 - wy) * (1.0 - wz));
        adj[b + nxp] += g * ((1.0 - wx) * wy * (1.0 - wz));
        adj[b + nxp + 1] += g * (wx * wy * (1.0 - wz));
        adj[b + sxy] += g * ((1.0 - wx) * (1.0 - wy) * wz);
        adj[b + sxy + 1] += g * (wx * (1.0 - wy) * wz);
        adj[b + sxy + nxp] += g * ((1.0 - wx) * wy * wz);
        adj[b + sxy + nxp + 1] += g * (wx * wy * wz);
      } else {
        double v00 = volp[b] * (1.0 - wx) + volp[b + 1] * wx;
        double v01 = volp[b + nxp] * (1.0 - wx) + volp[b + nxp + 1] * wx;
        double v10 = volp[b + sxy] * (1.0 - wx) + volp[b + sxy + 1] * wx;
        double v11 = volp[b + sxy + nxp] * (1.0 - wx) + volp[b + sxy + nxp + 1] * wx;
        double val = (v00 * (1.0 - wy) + v01 * wy) * (1.0 - wz) +
                     (v10 * (1.0 - wy) + v11 * wy) * wz;
        acc += val * seg;
      }
    }
    t += seg;
  }
  return acc;
}

int ora_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void ora_set_num_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* _kernels.py:160-171 (forward_parallel_2d). */
void ora_forward_parallel_2d(const double *volp, int nyp, int nxp, double sy,
                             double sx, const double *cos_a, const double *sin_a,
                             int n_ang, int n_det, double ds, double step,
                             double *out) {
  double half = (n_det - 1) / 2.0;
  long total = (long)n_ang * n_det;
#pragma omp parallel for schedule(dynamic, 64)
  for (long idx = 0; idx < total; ++idx) {
    long ia = idx / n_det;
    long j = idx % n_det;
    double ct = cos_a[ia], st = sin_a[ia];
    double t = (j - half) * ds;
    out[idx] = march_2d(volp, nyp, nxp, sy, sx, t * ct, t * st, -st, ct, step, NULL, 0.0);
  }
}

/* _kernels.py:174-195 (back_parallel_2d). */
void ora_back_parallel_2d(const double *sino, int n_ang, int n_det,
                          const double *cos_a, const double *sin_a, double ds,
                          int ny, int nx, double sy, double sx, double *out) {
  double half = (n_det - 1) / 2.0;
  double cy = (ny - 1) / 2.0, cx = (nx - 1) / 2.0;
  long total = (long)ny * nx;
#pragma omp parallel for schedule(static)
  for (long idx = 0; idx < total; ++idx) {
    long iy = idx / nx, ix = idx % nx;
    double x = (ix - cx) * sx;
    double y = (iy - cy) * sy;
    double acc = 0.0;
    for (int ia = 0; ia < n_ang; ++ia) {
      double t = x * cos_a[ia] + y * sin_a[ia];
      double f = t / ds + half;
      long j0 = (long)floor(f);
      double w = f - j0;
      if (0 <= j0 && j0 < n_det) acc += (1.0 - w) * sino[(long)ia * n_det + j0];
      if (0 <= j0 + 1 && j0 + 1 < n_det) acc += w * sino[(long)ia * n_det + j0 + 1];
    }
    out[idx] = acc;
  }
}

/* _kernels.py:198-216 (forward_fan_2d). */
static void fan_ray(double ct, double st, double sdd, double sid, double u,
                    double *sx_, double *sy_, double *dx, double *dy) {
  double srcx = sid * ct, srcy = sid * st;
  double pixx = -(sdd - sid) * ct - u * st;
  double pixy = -(sdd - sid) * st + u * ct;
  double ddx = pixx - srcx, ddy = pixy - srcy;
  double norm = sqrt(ddx * ddx + ddy * ddy);
  *sx_ = srcx; *sy_ = srcy; *dx = ddx / norm; *dy = ddy / norm;
}

void ora_forward_fan_2d(const double *volp, int nyp, int nxp, double sy,
                        double sx, const double *cos_a, const double *sin_a,
                        int n_ang, double sdd, double sid, int n_det, double ds,
                        double step, double *out) {
  double half = (n_det - 1) / 2.0;
  long total = (long)n_ang * n_det;
#pragma omp parallel for schedule(dynamic, 64)
  for (long idx = 0; idx < total; ++idx) {
    long ia = idx / n_det, j = idx % n_det;
    double px, py, dx, dy;
    fan_ray(cos_a[ia], sin_a[ia], sdd, sid, (j - half) * ds, &px, &py, &dx, &dy);
    out[idx] = march_2d(volp, nyp, nxp, sy, sx, px, py, dx, dy, step, NULL, 0.0);
  }
}

/* _kernels.py:219-251 (back_fan_2d). */
void ora_back_fan_2d(const double *sino, int n_ang, int n_det, const double *cos_a,
                     const double *sin_a, double sdd, double sid, double ds,
                     int ny, int nx, double sy, double sx, int weighted,
                     double *out) {
  double half = (n_det - 1) / 2.0;
  double cy = (ny - 1) / 2.0, cx = (nx - 1) / 2.0;
  long total = (long)ny * nx;
#pragma omp parallel for schedule(static)
  for (long idx = 0; idx < total; ++idx) {
    long iy = idx / nx, ix = idx % nx;
    double x = (ix - cx) * sx;
    double y = (iy - cy) * sy;
    double acc = 0.0;
    for (int ia = 0; ia < n_ang; ++ia) {
      double ct = cos_a[ia], st = sin_a[ia];
      double w = sid - x * ct - y * st;
      if (w <= TINY) continue;
      double u = sdd * (-x * st + y * ct) / w;
      double f = u / ds + half;
      long j0 = (long)floor(f);
      double fw = f - j0;
      double val = 0.0;
      if (0 <= j0 && j0 < n_det) val += (1.0 - fw) * sino[(long)ia * n_det + j0];
      if (0 <= j0 + 1 && j0 + 1 < n_det) val += fw * sino[(long)ia * n_det + j0 + 1];
      if (weighted) {
        double q = sid / w;
        val *= q * q;
      }
      acc += val;
    }
    out[idx] = acc;
  }
}

/* _kernels.py:254-278 (forward_cone_3d).  sources (V,3), minv (V,3,3). */
void ora_forward_cone_3d(const double *volp, int nzp, int nyp, int nxp, double sz,
                         double sy, double sx, const double *sources,
                         const double *minv, int n_views, int rows, int cols,
                         double step, double *out) {
  long total = (long)n_views * rows * cols;
#pragma omp parallel for schedule(dynamic, 256)
  for (long idx = 0; idx < total; ++idx) {
    long i = idx / ((long)rows * cols);
    long r = (idx / cols) % rows;
    long c = idx % cols;
    const double *m = minv + 9 * i;
    double dx = m[0] * c + m[1] * r + m[2];
    double dy = m[3] * c + m[4] * r + m[5];
    double dz = m[6] * c + m[7] * r + m[8];
    double norm = sqrt(dx * dx + dy * dy + dz * dz);
    out[idx] = march_3d(volp, nzp, nyp, nxp, sz, sy, sx, sources[3 * i],
                        sources[3 * i + 1], sources[3 * i + 2], dx / norm,
                        dy / norm, dz / norm, step, NULL, 0.0);
  }
}

/* _kernels.py:281-322 (back_cone_3d).  mats (V,3,4). */
void ora_back_cone_3d(const double *sino, int n_views, int rows, int cols,
                      const double *mats, double sid, int weighted, int nz,
                      int ny, int nx, double sz, double sy, double sx,
                      double *out) {
  double cz = (nz - 1) / 2.0, cy = (ny - 1) / 2.0, cx = (nx - 1) / 2.0;
  long total = (long)nz * ny * nx;
  long plane = (long)rows * cols;
#pragma omp parallel for schedule(static)
  for (long idx = 0; idx < total; ++idx) {
    long iz = idx / ((long)ny * nx);
    long iy = (idx / nx) % ny;
    long ix = idx % nx;
    double x = (ix - cx) * sx;
    double y = (iy - cy) * sy;
    double z = (iz - cz) * sz;
    double acc = 0.0;
    for (int i = 0; i < n_views; ++i) {
      const double *P = mats + 12 * i;
      double w = P[8] * x + P[9] * y + P[10] * z + P[11];
      if (w <= TINY) continue;
      double a = P[0] * x + P[1] * y + P[2] * z + P[3];
      double b = P[4] * x + P[5] * y + P[6] * z + P[7];
      double fc = a / w, fr = b / w;
      long c0 = (long)floor(fc), r0 = (long)floor(fr);
      double wc = fc - c0, wr = fr - r0;
      const double *s = sino + (long)i * plane;
      double val = 0.0;
      if (0 <= r0 && r0 < rows) {
        if (0 <= c0 && c0 < cols) val += (1.0 - wr) * (1.0 - wc) * s[r0 * cols + c0];
        if (0 <= c0 + 1 && c0 + 1 < cols) val += (1.0 - wr) * wc * s[r0 * cols + c0 + 1];
      }
      if (0 <= r0 + 1 && r0 + 1 < rows) {
        if (0 <= c0 && c0 < cols) val += wr * (1.0 - wc) * s[(r0 + 1) * cols + c0];
        if (0 <= c0 + 1 && c0 + 1 < cols) val += wr * wc * s[(r0 + 1) * cols + c0 + 1];
      }
      if (weighted) {
        double q = sid / w;
        val *= q * q;
      }
      acc += val;
    }
    out[idx] = acc;
  }
}

/* ---- exact transposes of the ray-driven forward operators (oracle for A^T) ---- */

/* Transpose of ora_forward_parallel_2d: adjp is the PADDED (ny+2, nx+2) output. */
void ora_forward_parallel_2d_transpose(const double *sino, int nyp, int nxp,
                                       double sy, double sx, const double *cos_a,
                                       const double *sin_a, int n_ang, int n_det,
                                       double ds, double step, double *adjp) {
  double half = (n_det - 1) / 2.0;
  memset(adjp, 0, sizeof(double) * (size_t)nyp * nxp);
  for (long idx = 0; idx < (long)n_ang * n_det; ++idx) {
    long ia = idx / n_det, j = idx % n_det;
    double ct = cos_a[ia], st = sin_a[ia];
    double t = (j - half) * ds;
    march_2d(NULL, nyp, nxp, sy, sx, t * ct, t * st, -st, ct, step, adjp, sino[idx]);
  }
}

void ora_forward_fan_2d_transpose(const double *sino, int nyp, int nxp, double sy,
                                  double sx, const double *cos_a,
                                  const double *sin_a, int n_ang, double sdd,
                                  double sid, int n_det, double ds, double step,
                                  double *adjp) {
  double half = (n_det - 1) / 2.0;
  memset(adjp, 0, sizeof(double) * (size_t)nyp * nxp);
  for (long idx = 0; idx < (long)n_ang * n_det; ++idx) {
    long ia = idx / n_det, j = idx % n_det;
    double px, py, dx, dy;
    fan_ray(cos_a[ia], sin_a[ia], sdd, sid, (j - half) * ds, &px, &py, &dx, &dy);
    march_2d(NULL, nyp, nxp, sy, sx, px, py, dx, dy, step, adjp, sino[idx]);
  }
}

void ora_forward_cone_3d_transpose(const double *sino, int nzp, int nyp, int nxp,
                                   double sz, double sy, double sx,
                                   const double *sources, const double *minv,
                                   int n_views, int rows, int cols, double step,
                                   double *adjp) {
  memset(adjp, 0, sizeof(double) * (size_t)nzp * nyp * nxp);
  for (long idx = 0; idx < (long)n_views * rows * cols; ++idx) {
    long i = idx / ((long)rows * cols);
    long r = (idx / cols) % rows;
    long c = idx % cols;
    const double *m = minv + 9 * i;
    double dx = m[0] * c + m[1] * r + m[2];
    double dy = m[3] * c + m[4] * r + m[5];
    double dz = m[6] * c + m[7] * r + m[8];
    double norm = sqrt(dx * dx + dy * dy + dz * dz);
    march_3d(NULL, nzp, nyp, nxp, sz, sy, sx, sources[3 * i], sources[3 * i + 1],
             sources[3 * i + 2], dx / norm, dy / norm, dz / norm, step, adjp,
             sino[idx]);
  }
}

/* Transpose of ora_back_cone_3d (voxel-driven) -- splats each voxel into the
 * sinogram with the same bilinear weights.  Serial. */
void ora_back_cone_3d_transpose(const double *vol, int n_views, int rows, int cols,
                                const double *mats, double sid, int weighted,
                                int nz, int ny, int nx, double sz, double sy,
                                double sx, double *sino) {
  double cz = (nz - 1) / 2.0, cy = (ny - 1) / 2.0, cx = (nx - 1) / 2.0;
  long plane = (long)rows * cols;
  memset(sino, 0, sizeof(double) * (size_t)n_views * plane);
  for (int i = 0; i < n_views; ++i) {
    const double *P = mats + 12 * i;
    double *s = sino + (long)i * plane;
    for (long idx = 0; idx < (long)nz * ny * nx; ++idx) {
      long iz = idx / ((long)ny * nx), iy = (idx / nx) % ny, ix = idx % nx;
      double x = (ix - cx) * sx, y = (iy - cy) * sy, z = (iz - cz) * sz;
      double w = P[8] * x + P[9] * y + P[10] * z + P[11];
      if (w <= TINY) continue;
      double a = P[0] * x + P[1] * y + P[2] * z + P[3];
      double b = P[4] * x + P[5] * y + P[6] * z + P[7];
      double fc = a / w, fr = b / w;
      long c0 = (long)floor(fc), r0 = (long)floor(fr);
      double wc = fc - c0, wr = fr - r0;
      double g = vol[idx];
      if (weighted) {
        double q = sid / w;
        g *= q * q;
      }
      if (0 <= r0 && r0 < rows) {
        if (0 <= c0 && c0 < cols) s[r0 * cols + c0] += g * ((1.0 - wr) * (1.0 - wc));
        if (0 <= c0 + 1 && c0 + 1 < cols) s[r0 * cols + c0 + 1] += g * ((1.0 - wr) * wc);
      }
      if (0 <= r0 + 1 && r0 + 1 < rows) {
        if (0 <= c0 && c0 < cols) s[(r0 + 1) * cols + c0] += g * (wr * (1.0 - wc));
        if (0 <= c0 + 1 && c0 + 1 < cols) s[(r0 + 1) * cols + c0 + 1] += g * (wr * wc);
      }
    }
  }
}

/* Exact transposes of the 2D voxel-driven back projectors (back_parallel_2d,
 * _kernels.py:174-195; back_fan_2d, :219-251): every pixel scatters its value
 * times the two linear-interpolation weights it gathers with (and the fan
 * distance weight) into the sinogram row of each angle.  Angles are
 * independent rows: parallel over angles, deterministic. */
void ora_back_parallel_2d_transpose(const double *img, int n_ang, int n_det, const double *cos_a,
                                    const double *sin_a, double ds, int ny, int nx, double sy,
                                    double sx, double *sino) {
  double half = (n_det - 1) / 2.0;
  double cy = (ny - 1) / 2.0, cx = (nx - 1) / 2.0;
#pragma omp parallel for schedule(static)
  for (int ia = 0; ia < n_ang; ++ia) {
    double *row = sino + (long)ia * n_det;
    for (int j = 0; j < n_det; ++j) row[j] = 0.0;
    for (long idx = 0; idx < (long)ny * nx; ++idx) {
      long iy = idx / nx, ix = idx % nx;
      double x = (ix - cx) * sx, y = (iy - cy) * sy;
      double f = (x * cos_a[ia] + y * sin_a[ia]) / ds + half;
      long j0 = (long)floor(f);
      double w = f - j0, g = img[idx];
      if (0 <= j0 && j0 < n_det) row[j0] += (1.0 - w) * g;
      if (0 <= j0 + 1 && j0 + 1 < n_det) row[j0 + 1] += w * g;
    }
  }
}

void ora_back_fan_2d_transpose(const double *img, int n_ang, int n_det, const double *cos_a,
                               const double *sin_a, double sdd, double sid, double ds, int ny,
                               int nx, double sy, double sx, int weighted, double *sino) {
  double half = (n_det - 1) / 2.0;
  double cy = (ny - 1) / 2.0, cx = (nx - 1) / 2.0;
#pragma omp parallel for schedule(static)
  for (int ia = 0; ia < n_ang; ++ia) {
    double *row = sino + (long)ia * n_det;
    double ct = cos_a[ia], st = sin_a[ia];
    for (int j = 0; j < n_det; ++j) row[j] = 0.0;
    for (long idx = 0; idx < (long)ny * nx; ++idx) {
      long iy = idx / nx, ix = idx % nx;
      double x = (ix - cx) * sx, y = (iy - cy) * sy;
      double w = sid - x * ct - y * st;
      if (w <= TINY) continue;
      double f = sdd * (-x * st + y * ct) / w / ds + half;
      long j0 = (long)floor(f);
      double fw = f - j0, g = img[idx];
      if (weighted) {
        double q = sid / w;
        g *= q * q;
      }
      if (0 <= j0 && j0 < n_det) row[j0] += (1.0 - fw) * g;
      if (0 <= j0 + 1 && j0 + 1 < n_det) row[j0 + 1] += fw * g;
    }
  }
}
