/*
 * tk_b200.h -- C ABI of the B200 (sm_100a) CT-operator library (libtkb200.so).
 *
 * Drop-in boundary for the reference's projector kernel layer
 * (/root/reference/pkg/src/tomokit/_kernels.py) and its FFT row filter
 * (/root/reference/pkg/src/tomokit/filters.py).  Conventions follow the
 * reference exactly (see _kernels.py:9-16, grids.py:8-11):
 *   - world coordinate of index i on an axis with n samples, spacing s:
 *     (i - (n-1)/2) * s ; volumes are C-order (y,x) / (z,y,x);
 *     sinograms (view,u) / (view,v,u) with u the fastest axis;
 *   - forward operators integrate the zero-extended bi/trilinear interpolant
 *     with midpoint sampling at `step` (last partial step exact), in value*mm;
 *   - back operators are voxel-driven linear/bilinear gathers, optionally
 *     weighted by (sid/w)^2.
 *
 * Memory: every float* grid argument is a DEVICE pointer (fp32, C-contiguous).
 * Per-view geometry (angles as cos/sin, projection matrices, sources, M^-1) is
 * passed as HOST float64 arrays -- exactly the arrays the reference computes on
 * the host (projectors.py:106-248) -- and packed/uploaded by the library.
 * `stream` is a cudaStream_t (NULL = legacy default stream).  All calls are
 * stream-ordered and asynchronous with respect to the host; scratch memory is
 * stream-ordered (cudaMallocAsync) and released before return.  Outputs are
 * fully overwritten (unless an `accumulate` flag says otherwise); inputs are
 * never modified.  Unlike the reference, volumes are passed UNPADDED: the
 * one-voxel zero margin of projectors.py:26-29 is applied inside the library.
 *
 * Every function returns 0 on success, TK_ERR_ARG for an invalid argument,
 * TK_ERR_CUDA for a CUDA error; tk_last_error() returns the thread's message.
 */
#ifndef TK_B200_H
#define TK_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TK_OK 0
#define TK_ERR_ARG 1
#define TK_ERR_CUDA 2

/* Library identity and diagnostics. */
int tk_version(void);                 /* major*10000 + minor*100 + patch */
const char *tk_last_error(void);      /* thread-local; "" when no error */
int tk_device_info(int *sm_major, int *sm_minor, int *sm_count);
/* Number of kernel launches issued by this library since load (all threads). */
unsigned long long tk_launch_count(void);
/* The texture-gather kernels copy grids into pooled block-linear CUDA arrays
 * that are kept between calls (stream-ordered reuse).  Bytes held / free all
 * idle ones. */
unsigned long long tk_cached_bytes(void);
int tk_release_cached_memory(void);

/* ---- parallel-beam 2D ------------------------------------------------------
 * replaces _kernels.forward_parallel_2d (_kernels.py:160-171), called from
 * projectors.forward_project_parallel_2d (projectors.py:106-123).
 * vol (ny,nx) device; cos_a/sin_a host float64[n_ang]; out (n_ang,n_det). */
int tk_forward_parallel_2d(const float *vol, int ny, int nx, double sy, double sx,
                           const double *cos_a, const double *sin_a, int n_ang,
                           int n_det, double ds, double step, float *out,
                           void *stream);
/* replaces _kernels.back_parallel_2d (_kernels.py:174-195),
 * projectors.back_project_parallel_2d (projectors.py:126-142). */
int tk_back_parallel_2d(const float *sino, int n_ang, int n_det,
                        const double *cos_a, const double *sin_a, double ds,
                        int ny, int nx, double sy, double sx, float *out,
                        void *stream);

/* ---- fan-beam 2D -----------------------------------------------------------
 * replaces _kernels.forward_fan_2d (_kernels.py:198-216). */
int tk_forward_fan_2d(const float *vol, int ny, int nx, double sy, double sx,
                      const double *cos_a, const double *sin_a, int n_ang,
                      double sdd, double sid, int n_det, double ds, double step,
                      float *out, void *stream);
/* replaces _kernels.back_fan_2d (_kernels.py:219-251). */
int tk_back_fan_2d(const float *sino, int n_ang, int n_det, const double *cos_a,
                   const double *sin_a, double sdd, double sid, double ds, int ny,
                   int nx, double sy, double sx, int weighted, float *out,
                   void *stream);

/* ---- cone-beam 3D ----------------------------------------------------------
 * replaces _kernels.forward_cone_3d (_kernels.py:254-278) as called from
 * projectors.forward_project_cone_3d (projectors.py:205-225).
 * vol (nz,ny,nx) device; sources host float64 (V,3); minv host float64 (V,3,3)
 * (= projectors._cone_rays, projectors.py:191-202); out (V,rows,cols). */
int tk_forward_cone_3d(const float *vol, int nz, int ny, int nx, double sz,
                       double sy, double sx, const double *sources,
                       const double *minv, int n_views, int rows, int cols,
                       double step, float *out, void *stream);
/* Which forward kernel tk_forward_cone_3d runs for this scan (host-only query,
 * no device work): 1 = the z-mirror-pair kernel (every view z-mirror
 * symmetric -- circular orbits with the principal row at (R-1)/2 -- and the
 * volume fits its layout), 0 = the general ray-per-thread kernel. */
/* View-sharded forward projection fused with the multi-GPU row-band exchange
 * (no reference counterpart; distributed.py): ray (v, r, c) of these n_views views is
 * stored into every destination h whose detector row band [r0[h], r1[h]) holds row r, at
 * dest[h] + ((view_offset + v) * band_pitch_rows + (r - r0[h])) * cols + c.  dest[h] may be
 * a peer GPU's buffer (CUDA IPC / symmetric memory over NVLink): the stores are the
 * exchange, issued ray by ray as the projection runs.  1..16 destinations. */
int tk_forward_cone_3d_bands(const float *vol, int nz, int ny, int nx, double sz, double sy,
                             double sx, const double *sources, const double *minv, int n_views,
                             int rows, int cols, double step, int view_offset, int n_dest,
                             float *const *dest, const int *r0, const int *r1,
                             int band_pitch_rows, void *stream);
int tk_forward_cone_3d_path(const double *sources, const double *minv, int n_views, int rows,
                            int cols, int nz, int ny, int nx);
/* Forward-projection plan (no reference counterpart): the per-volume
 * preprocessing of tk_forward_cone_3d (the zero-margin, z-fastest coefficient
 * cells of the volume) done once, then any number of view blocks projected from
 * it -- e.g. view chunks whose D2H copies overlap the next chunk's kernel.  The
 * cells are built on the first tk_fp_plan_project call, on that call's stream,
 * from `vol`: the volume must stay allocated and unchanged until then.  *plan is
 * an opaque handle; destroy frees it stream-ordered on `stream` (the caller
 * orders other streams' uses before that). */
int tk_fp_plan_create(const float *vol, int nz, int ny, int nx, double sz, double sy,
                      double sx, void **plan, void *stream);
int tk_fp_plan_project(void *plan, const double *sources, const double *minv,
                       int n_views, int rows, int cols, double step, float *out,
                       void *stream);
int tk_fp_plan_destroy(void *plan, void *stream);
/* replaces _kernels.back_cone_3d (_kernels.py:281-322) as called from
 * projectors.back_project_cone_3d (projectors.py:228-248).
 * sino (V,rows,cols) device; mats host float64 (V,3,4); out (nz,ny,nx). */
int tk_back_cone_3d(const float *sino, int n_views, int rows, int cols,
                    const double *mats, double sid, int weighted, int nz, int ny,
                    int nx, double sz, double sy, double sx, float *out,
                    void *stream);
/* Sharded variant of tk_back_cone_3d (no reference counterpart; multi-GPU
 * z-slab / view-chunk decomposition).  Computes the voxels with global z index
 * in [z_begin, z_begin+z_count) of the (nz,ny,nx) grid into out (z_count,ny,nx),
 * reading a detector row band: `sino` holds rows [row_begin, row_begin+band_rows)
 * of every view (V, band_rows, cols); rows outside the band read as zero.
 * accumulate != 0 adds into out instead of overwriting it. */
int tk_back_cone_3d_ex(const float *sino, int n_views, int rows, int cols,
                       int row_begin, int band_rows, const double *mats,
                       double sid, int weighted, int nz, int ny, int nx,
                       double sz, double sy, double sx, int z_begin, int z_count,
                       int accumulate, float *out, void *stream);

/* ---- matched adjoints (exact transposes; not in the reference, which pairs
 * A with the unmatched voxel-driven B, autodiff.py:1-19) ------------------------
 * Scatter kernels (fp32 atomics: results are deterministic only up to fp32
 * summation order).  out is overwritten. */
int tk_forward_cone_3d_adjoint(const float *sino, int n_views, int rows, int cols,
                               const double *sources, const double *minv,
                               int nz, int ny, int nx, double sz, double sy,
                               double sx, double step, float *vol_out,
                               void *stream);
/* As tk_forward_cone_3d_adjoint; deterministic = 1 accumulates in fixed point with
 * integer atomics (scale 2^e from a magnitude pass, the same scatter of |sino|; two
 * components per 64-bit word): bit-reproducible, ~2.7x the fp32 time. */
int tk_forward_cone_3d_adjoint_ex(const float *sino, int n_views, int rows, int cols,
                                  const double *sources, const double *minv, int nz, int ny,
                                  int nx, double sz, double sy, double sx, double step,
                                  int deterministic, float *vol_out, void *stream);
int tk_back_cone_3d_adjoint(const float *vol, int nz, int ny, int nx, double sz,
                            double sy, double sx, const double *mats, double sid,
                            int weighted, int n_views, int rows, int cols,
                            float *sino_out, void *stream);
int tk_forward_parallel_2d_adjoint(const float *sino, int n_ang, int n_det,
                                   const double *cos_a, const double *sin_a,
                                   double ds, double step, int ny, int nx,
                                   double sy, double sx, float *vol_out,
                                   void *stream);
int tk_forward_fan_2d_adjoint(const float *sino, int n_ang, int n_det,
                              const double *cos_a, const double *sin_a,
                              double sdd, double sid, double ds, double step,
                              int ny, int nx, double sy, double sx, float *vol_out,
                              void *stream);
/* Exact transposes B^T of tk_back_parallel_2d / tk_back_fan_2d (the matched adjoint
 * of the reference's voxel-driven 2D back projectors, _kernels.py:174-251; the
 * reference's own VJP of back projection is the paired A, autodiff.py:65-68).
 * sino_out (n_ang, n_det) is overwritten; weighted = 1 applies (sid / w)^2 (fan). */
int tk_back_parallel_2d_adjoint(const float *img, int ny, int nx, double sy, double sx,
                                const double *cos_a, const double *sin_a, int n_ang,
                                int n_det, double ds, float *sino_out, void *stream);
int tk_back_fan_2d_adjoint(const float *img, int ny, int nx, double sy, double sx,
                           const double *cos_a, const double *sin_a, int n_ang, double sdd,
                           double sid, int n_det, double ds, int weighted, float *sino_out,
                           void *stream);

/* ---- FFT row filter (filters.py:136-171, 204-211) ---------------------------
 * For each of n_rows rows of `width` samples (row r belongs to detector row
 * (r % det_rows)): optional obliquity pre-weight sdd/sqrt(sdd^2+u^2+v^2)
 * (u,v metric detector offsets with pitches du,dv; disabled when sdd <= 0),
 * zero-pad to n_pad (power of two >= 2*width), multiply DFT bin k by
 * half_weights[min(k, n_pad-k)] (host float64[n_pad/2+1]), inverse transform,
 * crop to width and scale by `scale` (the filter's detector_spacing).
 * in and out may alias. */
int tk_fft_filter_rows(const float *in, long long n_rows, int width, int det_rows,
                       const double *half_weights, int n_pad, double scale,
                       double sdd, double du, double dv, float *out,
                       void *stream);

/* Row-band variant for z-slab sharding: the buffer holds `band_rows` detector
 * rows starting at detector row `row_offset` of a `det_rows`-row detector
 * (buffer row r is detector row (r % band_rows) + row_offset, which sets the v
 * coordinate of the pre-weight). */
int tk_fft_filter_rows_ex(const float *in, long long n_rows, int width, int band_rows,
                          int row_offset, int det_rows, const double *half_weights,
                          int n_pad, double scale, double sdd, double du, double dv,
                          float *out, void *stream);

/* ---- helpers --------------------------------------------------------------- */
/* out[i] = in[i] * scale (fp32), n elements; in/out may alias. */
int tk_scale(const float *in, long long n, double scale, float *out, void *stream);

/* ---- sinogram degradation simulators (reference artifacts.py:50-211) ----
 * Elementwise / small-stencil kernels on device sinograms (n_views, rows, cols)
 * (rows = 1 for 2D).  Noise comes from a counter-based Philox4x32-10 stream
 * per (seed, view), indexed by texel: reproducible for a seed, independent of
 * launch configuration; the distributions are the contract (artifacts.py:5-7).
 * out may not alias sino. */
/* the per-view integer offsets tk_detector_jitter draws, uniform in [-max, max] (host) */
int tk_jitter_shifts(unsigned long long seed, int n_views, int max_shift, int *shifts_out);
/* add_detector_jitter (artifacts.py:50-66): shift each view by its offset along
 * u (axis_v = 0) or v (axis_v = 1), zero-filling the vacated strip */
int tk_detector_jitter(const float *sino, int n_views, int rows, int cols, int axis_v, int max_shift,
                       unsigned long long seed, float *out, void *stream);
/* add_poisson_noise (artifacts.py:69-93): transmission = 1: -ln(max(Poisson(i0 e^-p), 1) / i0);
 * transmission = 0: Poisson(p) (direct mode) */
int tk_poisson_noise(const float *sino, int n_views, long long view_size, double i0, int transmission,
                     unsigned long long seed, float *out, void *stream);
/* add_gaussian_noise (artifacts.py:96-105): p + mean + std N(0, 1) */
int tk_gaussian_noise(const float *sino, int n_views, long long view_size, double mean, double std,
                      unsigned long long seed, float *out, void *stream);
/* add_ring_artifact (artifacts.py:108-146): host columns[n_columns]; views [start, end);
 * zero = 1 clears them, zero = 0 multiplies by factor; everything else copied bit-exact */
int tk_ring_artifact(const float *sino, int n_views, int rows, int cols, const int *columns, int n_columns,
                     int start, int end, int zero, double factor, float *out, void *stream);
/* add_gantry_motion_blur (artifacts.py:183-211): zero-padded 2D convolution of view i with
 * the host float64 kernel kernels[i][2 half + 1][2 half + 1] (rows: v, columns: u) */
int tk_gantry_blur(const float *sino, int n_views, int rows, int cols, const double *kernels, int half,
                   float *out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* TK_B200_H */
