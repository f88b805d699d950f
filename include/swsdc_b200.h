/*
 * swsdc_b200.h -- C ABI of the B200 (sm_100a) MLSDC-SH hot path.
 *
 * Drop-in boundary for the reference package `swsdc` (/root/reference/pkg/src/swsdc).
 * The reference has no FFI: its boundary is duck-typed Python objects.  Each
 * entry point below replaces one reference method; the Python mirror in
 * paper_1805_07923_b200/ (spharm.py, swe.py, implicit.py, sdc.py, mlsdc.py)
 * binds these symbols with ctypes and keeps the reference's names, argument
 * meaning and exceptions.
 *
 * Conventions
 *   - All array arguments are DEVICE pointers owned by the caller.
 *   - Spectral arrays: complex128 (interleaved re, im doubles), dense
 *     triangular layout [r][s], (R+1) x (R+1) per field, zeros for s < r
 *     (spharm.py:6-10).  A prognostic state is 3 such fields
 *     (phi_prime, zeta, delta) back to back (swe.py:44-58).
 *   - Grid arrays: float64 (n_lon, n_lat), longitude-major, latitudes ascending
 *     in mu (spharm.py:3-5).
 *   - `batch` independent fields / states are contiguous.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *     stream-ordered and asynchronous; a plan's scratch workspace serialises
 *     calls that share the plan, so use one plan per concurrent stream.
 *   - Return value: 0 ok, 1 usage error (-> ValueError), 2 numerical error
 *     (-> RuntimeError), 3 CUDA error.  swsdc_last_error() describes the last
 *     failure of the calling thread.
 */
#ifndef SWSDC_B200_H
#define SWSDC_B200_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct swsdc_plan swsdc_plan;

/* Model constants in the order (radius, omega, gravity, nu, h_bar); phi_bar = gravity * h_bar
 * (swe.py:20-41). */
typedef struct swsdc_params {
  double radius, omega, gravity, nu, h_bar;
} swsdc_params;

const char* swsdc_last_error(void);
const char* swsdc_version(void);

/* TransformPlan.__init__ (spharm.py:189-206): validates the truncation, builds
 * the device recurrence tables, checkpoint seeds and FFT twiddles.  mu, w are
 * HOST arrays of the n_lat Gauss nodes / weights (spharm.py:52-86). */
int swsdc_plan_create(int truncation, int n_lon, int n_lat, const double* mu, const double* w,
                      swsdc_plan** out);
int swsdc_plan_destroy(swsdc_plan* plan);
/* Plan options: key 1 = force the large-n_lon F_E path (grids through HBM) even when the
 * fused shared-memory grid kernel fits (used by the tests to check both paths). */
int swsdc_plan_config(swsdc_plan* plan, int key, int value);
/* Pre-size the scratch workspace for up to `fields` simultaneous fields (so no
 * allocation happens later, e.g. during CUDA graph capture).  Workspaces a stream
 * capture has used are pinned: later growth allocates fresh buffers and keeps the
 * pinned ones alive until swsdc_plan_destroy, so captured graphs stay valid. */
int swsdc_plan_reserve(swsdc_plan* plan, int fields);

/* TransformPlan.synthesize (spharm.py:258-260); coefficients at truncation
 * r_in <= R are zero-padded (spharm.py:242-250). */
int swsdc_synthesize(swsdc_plan* plan, const double* coeffs, int r_in, int batch, double* grid,
                     void* stream);
/* TransformPlan.analyze (spharm.py:254-256). */
int swsdc_analyze(swsdc_plan* plan, const double* grid, int batch, double* coeffs, void* stream);
/* TransformPlan.synthesize_pair_cos_gradient (spharm.py:262-279), unit sphere. */
int swsdc_synthesize_uv(swsdc_plan* plan, const double* psi, const double* chi, int r_in, int batch,
                        double* u, double* v, void* stream);
/* TransformPlan.analyze_vector_div_curl (spharm.py:281-300), unit sphere. */
int swsdc_analyze_divcurl(swsdc_plan* plan, const double* u, const double* v, int batch,
                          double* div, double* curl, void* stream);

/* ShallowWaterRHS.eval_f_e (swe.py:251-279) for `batch` states. */
int swsdc_eval_fe(swsdc_plan* plan, const swsdc_params* params, int include_nonlinear,
                  const double* state, int batch, double* out, void* stream);
/* m-sharding (multi-GPU).  swsdc_set_row_filter(P, rank) makes every
 * spectral-space kernel (solve, F_I, combine, resize, sweep node, analysis, F_E assembly)
 * process only rows r with r % P == rank ((1, 0) = all rows).  The F_E pipeline is then
 * run in stages with caller-owned exchange buffers so the caller can all-to-all between
 * them: eo = [batch][5][R+1][ceil(J/2)][E.re,E.im,O.re,O.im] (rows of this rank),
 * x = fragment-native analysis input (layout: swsdc_fe_layout) for latitude pairs
 * [jh_begin, jh_end) and all rows. */
int swsdc_set_row_filter(int mod, int rank);
int swsdc_fe_layout(swsdc_plan* plan, int include_nonlinear, int batch, long long* eo_doubles,
                    long long* x_doubles, int* x_nc, int* x_jh4);
int swsdc_fe_synthesis(swsdc_plan* plan, const swsdc_params* params, const double* state, int batch,
                       double* eo, void* stream);
int swsdc_fe_grid(swsdc_plan* plan, const swsdc_params* params, int include_nonlinear,
                  const double* eo, int batch, int jh_begin, int jh_end, double* x, void* stream);
int swsdc_fe_analysis(swsdc_plan* plan, const swsdc_params* params, int include_nonlinear,
                      const double* x, int batch, double* out, void* stream);

/* ShallowWaterRHS.eval_f_i / eval_l_g (swe.py:206-217, 246-249). */
int swsdc_eval_fi(int truncation, const swsdc_params* params, const double* state, int batch,
                  double* out, void* stream);
/* implicit.solve_implicit (implicit.py:31-49): (I - beta F_I) theta = b.  Returns 1
 * for beta < 0 and 2 when any 2x2 determinant is <= 0. */
int swsdc_solve_implicit(int truncation, const swsdc_params* params, double beta, const double* b,
                         int batch, double* out, void* stream);

/* out[i] = sum_k w[k] * x[k][i] over `count` doubles, n <= 32
 * (sdc._combine sdc.py:211-220 and PrognosticState algebra swe.py:77-102). */
int swsdc_combine(int n, const double* const* x, const double* w, long long count, double* out,
                  void* stream);
/* out = sum_k w[k] * resize(x[k], r_in[k] -> r_out) over `nmat` spectral matrices per input,
 * n <= 32: restriction (Lagrange rows + truncate, mlsdc.py:83-88), interpolation (pad +
 * Lagrange rows, mlsdc.py:90-95) and the FAS combination (mlsdc.py:113-124) in one launch. */
int swsdc_spec_combine(int n, const double* const* x, const double* w, const int* r_in, int r_out,
                       long long nmat, double* out, void* stream);
/* nout (<= 16) independent spec_combine sums in one launch: output o takes the next
 * nterms[o] entries of x / w / r_in (<= 96 terms in total); outputs may update one of
 * their own inputs in place (Step D of mlsdc_iteration, mlsdc.py:226-238), but no
 * output may be another output's input.  Used for the restriction, FAS and
 * interpolation groups of an MLSDC iteration (mlsdc.py:83-124).  ext (nullable): per output,
 * rows and columns above ext[o] are left untouched -- for in-place outputs whose other terms
 * are all at truncation <= ext[o] (x += padded coarse correction), only that block changes. */
int swsdc_spec_combine_multi(int nout, const int* nterms, const double* const* x, const double* w,
                             const int* r_in, int r_out, long long nmat, double* const* outs,
                             const int* ext, void* stream);
/* dst = src over n doubles and *bad = (any value non-finite): the stepper's per-step state
 * copy and finiteness check (harness.py:257) in one pass; *bad is cleared first. */
/* m-sharding exchange packing (distributed.py, exchange_eo / exchange_x): for the array
 * arr[outer][rows][cols][inner] (doubles) and nblocks (<= 64) blocks b -- rows row0[b] +
 * k row_step[b] (k < nrows[b]), columns [col0[b], col1[b]) -- gather them into the contiguous
 * buffer buf, block after block as [b][outer][k][col][inner] (scatter = 0), or scatter buf
 * back into arr (scatter = 1).  One launch instead of one strided copy per peer. */
int swsdc_exchange_blocks(double* arr, long long outer, long long rows, long long cols,
                          long long inner, int nblocks, const int* row0, const int* row_step,
                          const int* nrows, const int* col0, const int* col1, double* buf,
                          int scatter, void* stream);
int swsdc_copy_finite(const double* src, double* dst, long long n, int* bad, void* stream);
/* One SDC node update (sdc.py:196-206): b = sum_k w[k] x[k] (states at truncation R),
 * theta = solve_implicit(b, beta) (implicit.py:31-49), f_i = eval_f_i(theta)
 * (swe.py:206-217), for `batch` states.  Same status rules as swsdc_solve_implicit. */
int swsdc_sweep_node(int truncation, const swsdc_params* params, double beta, int n,
                     const double* const* x, const double* w, int batch, double* theta,
                     double* f_i, void* stream);
/* spharm.truncate / spharm.pad (spharm.py:331-349) over `nmat` (R+1)^2 matrices. */
int swsdc_resize(const double* in, int r_in, double* out, int r_out, long long nmat, void* stream);
/* spharm.laplacian / spharm.inv_laplacian (spharm.py:313-328) over `nmat` (R+1)^2
 * matrices: multiply (inverse = 0) or divide (inverse = 1, s = 0 column set to 0) by
 * -s(s+1)/radius^2; in == out allowed.  1 (usage) if radius <= 0. */
int swsdc_laplacian(const double* in, double* out, int truncation, long long nmat, double radius,
                    int inverse, void* stream);

/* Upload of `nmat` dense (R+1)^2 spectral matrices from page-locked host memory
 * (cudaHostAlloc / cudaHostRegister) to device `out`: only the s >= r triangle the
 * reference layout populates crosses PCIe (zero-copy reads); the device copy's lower
 * triangle is written as zeros.  The host-input half of TransformPlan.synthesize
 * (spharm.py:258-260) for host arrays; 1 when `host` is not page-locked. */
int swsdc_upload_coeffs(const double* host, int truncation, long long nmat, double* out,
                        void* stream);

/* Host-only half of the packed upload (SWSDC_UPLOAD_MODE=2): the s >= r triangles of
 * `nmat` dense (R+1)^2 host matrices, row after row, into `packed`
 * (nmat (R+1)(R+2)/2 complex values), by the library's pool of packing threads; returns
 * when done.  swsdc_upload_coeffs in that mode runs this asynchronously into a
 * page-locked staging buffer, gates the stream on it with a stream memory operation,
 * moves the buffer with one contiguous copy-engine transfer (the only kind that runs
 * PCIe full duplex next to a download) and expands it on the device.  No device needed. */
int swsdc_pack_triangles(const double* dense, int truncation, long long nmat, double* packed);

/* Download of `nmat` dense (R+1)^2 spectral matrices from device `dev` into page-locked
 * host memory by zero-copy stores.  write_lower = 1 writes the full dense matrices (the
 * reference's analyze result, spharm.py:254-256); write_lower = 0 guarantees only the s >= r
 * triangle: each entry below it is either left untouched or receives the device's value
 * (~half the PCIe bytes, for callers streaming results into a reused, zero-initialised
 * buffer, where either way it holds the reference's zero). */
int swsdc_download_coeffs(const double* dev, int truncation, long long nmat, double* host,
                          int write_lower, void* stream);

/* Launch accounting / stage timing (bench.py): number of kernels launched by
 * this library so far; per-stage CUDA-event timing on/off (clears records);
 * collect "stage<TAB>launches<TAB>total_ms" lines, returns bytes needed. */
long long swsdc_launch_count(void);
int swsdc_profile_enable(int on);
int swsdc_profile_collect(char* buf, int buflen);
/* FP64 FMA throughput probe (TFLOP/s) on the current device: the roofline
 * denominator bench.py measures live. */
int swsdc_probe_fp64(int reps, double* tflops);

#ifdef __cplusplus
}
#endif

#endif /* SWSDC_B200_H */
