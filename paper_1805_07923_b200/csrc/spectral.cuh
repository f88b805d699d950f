// Launch interfaces of the spectral-space kernels (spectral.cu).
#pragma once
#include "common.cuh"

namespace swsdc {

struct ModelConsts {
  double radius, omega, gravity, nu, h_bar, phi_bar;
};

// Rows r with r % mod == rank are processed (m-sharding, cyclic in r); other
// rows are neither read nor written.  {1, 0} = all rows.
struct RowFilter {
  int mod, rank;
};
RowFilter current_row_filter();

constexpr int kMaxCombine = 32;
struct CombineArgs {
  const double* x[kMaxCombine];
  double w[kMaxCombine];
  double* out;
  int n;
};

int launch_finalize_swe(const PlanDev& P, const double2* Y, long long y_mstride, int ldy,
                        double2* out, long long out_mstride, bool nonlin, double radius,
                        int nmembers, cudaStream_t st, RowFilter rf = {1, 0});
int launch_finalize_divcurl(const PlanDev& P, const double2* Y, long long y_mstride, int ldy,
                            double2* div, double2* curl, int nmembers, cudaStream_t st);
int launch_eval_fi(int R, const ModelConsts& c, const double2* x, double2* out, long long nmat,
                   cudaStream_t st);
int launch_solve(int R, const ModelConsts& c, double beta, const double2* b, double2* out,
                 long long nmat, cudaStream_t st);
int launch_combine(const CombineArgs& a, long long count, cudaStream_t st);

// Weighted sum of spectral states with per-input truncation, written at
// truncation rout (zero-padded / truncated): out = sum_k w_k resize(x_k).
struct SpecCombineArgs {
  const double2* x[kMaxCombine];
  double w[kMaxCombine];
  int rin[kMaxCombine];
  int n;
  double2* out;
  int rout;
};
int launch_spec_combine(const SpecCombineArgs& a, long long nmat, cudaStream_t st);
// Several independent weighted sums in one launch: output o (< nout) is
// sum over terms [off[o], off[o+1]) of w_k * resize(x_k, rin_k -> rout).
constexpr int kMultiOut = 16;
constexpr int kMultiTerms = 96;
struct MultiCombineArgs {
  const double2* x[kMultiTerms];
  double w[kMultiTerms];
  int rin[kMultiTerms];
  int off[kMultiOut + 1];
  double2* out[kMultiOut];
  int ext[kMultiOut];      // rows/columns > ext are left as they are (in-place outputs
                           // whose other terms are all coarser: x += padded correction)
  int nout;
  int rout;
};
int launch_spec_combine_multi(const MultiCombineArgs& a, long long nmat, cudaStream_t st);
// One sweep node (sdc.py:196-206 fused): b = sum_k w_k x_k (all at R);
// theta = solve(b, beta); fi = L_G(theta).  nstates = states per input.
int launch_sweep_node(int R, const ModelConsts& c, double beta, const SpecCombineArgs& a,
                      double2* theta, double2* fi, long long nstates, cudaStream_t st);
int launch_upload_triangle(const double2* host, double2* out, int R, long long nmat,
                           cudaStream_t st);
// hostpack.cu: host-packed triangles, one contiguous copy-engine transfer, device expansion
bool packed_upload_available();
int pack_triangles_host(const double2* dense, int R, long long nmat, double2* packed);
int launch_upload_packed(const double2* host, double2* out, int R, long long nmat, cudaStream_t st);
int launch_download_triangle(const double2* dev, double2* host, int R, long long nmat,
                             int write_lower, cudaStream_t st);
constexpr int kMaxExBlocks = 64;
struct ExchangeBlocks {
  long long rows, cols, C;            // array dims after the outer one: [A][rows][cols][C]
  int nb;
  int row0[kMaxExBlocks], row_step[kMaxExBlocks], nrows[kMaxExBlocks];
  int col0[kMaxExBlocks], col1[kMaxExBlocks];
  long long off[kMaxExBlocks + 1];    // doubles before block b in the buffer
};
int launch_exchange_blocks(const ExchangeBlocks& e, double* arr, double* buf, int scatter,
                           cudaStream_t st);
int launch_copy_finite(const double* src, double* dst, long long n, int* bad, cudaStream_t st);
int launch_zero_lower(double2* out, int R, long long nmat, cudaStream_t st);
int launch_resize(const double2* in, int rin, double2* out, int rout, long long nmat,
                  cudaStream_t st);
int launch_laplacian(const double2* in, double2* out, int R, long long nmat, double radius,
                     int inverse, cudaStream_t st);

}  // namespace swsdc
