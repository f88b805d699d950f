// Spectral-space kernels: O(T) per field, HBM-bound elementwise work.
//
//   finalize_swe      assembly of F_E from the analysed vectors incl. the
//                     H-shift sum_j H_s y_j = (s+1) eps_s Y_{s-1} - s eps_{s+1} Y_{s+1}
//                     and -lambda_s * analyze(KE)     (swe.py:261-279, spharm.py:171-178)
//   finalize_divcurl  analyze_vector_div_curl assembly (spharm.py:294-300)
//   eval_fi           L_G: gravity-wave coupling + diffusion (swe.py:206-217)
//   solve_implicit    per-(r, s) 2x2 + scalar closed form (implicit.py:31-49)
//   combine           sum_k w_k x_k (sdc.py:211-220, PrognosticState algebra swe.py:77-102)
//   resize            truncate / pad (spharm.py:331-349)
//   laplacian         laplacian / inv_laplacian (spharm.py:313-328)
//   sweep_rhs         b = theta0 + sum_j c_j F_j + ... (sdc.py:185-202), fused
#include <algorithm>
#include <cstdlib>
#include "common.cuh"
#include "spectral.cuh"

namespace swsdc {

static thread_local RowFilter g_row_filter{1, 0};
RowFilter current_row_filter() { return g_row_filter; }
void set_row_filter(int mod, int rank) { g_row_filter = RowFilter{mod, rank}; }

namespace {

__device__ __forceinline__ double lam_of(int s, double radius) {
  // spharm.py:307-310  -s (s+1) / a^2
  return (-(double)s * (s + 1.0)) / (radius * radius);
}

__device__ __forceinline__ double2 hshift(const double2* Yv, const double* eps_r, int r, int s) {
  // (s+1) eps_s Y_{s-1} - s eps_{s+1} Y_{s+1}; eps_r == 0 so the first term is absent at s == r
  const double2 up = Yv[s + 1];
  const double cu = s * eps_r[s + 1];
  double2 out = make_double2(-cu * up.x, -cu * up.y);
  if (s > r) {
    const double2 dn = Yv[s - 1];
    const double cd = (s + 1.0) * eps_r[s];
    out.x += cd * dn.x;
    out.y += cd * dn.y;
  }
  return out;
}

// Grid (s blocks, R + 1 rows, members): one row (m, r) per y/z coordinate,
// degrees s across x -- no per-element index division.
__global__ void finalize_swe_kernel(PlanDev P, const double2* Y, long long y_mstride, int ldy,
                                    double2* out, long long out_mstride, int nonlin,
                                    double radius, int nmembers, RowFilter rf) {
  pdl_wait();
  pdl_trigger();
  const int R = P.R;
  const int s = blockIdx.x * blockDim.x + threadIdx.x, r = blockIdx.y, m = blockIdx.z;
  if (s > R || r % rf.mod != rf.rank) return;
  (void)nmembers;
  const long long plane = (long long)(R + 1) * (R + 1);
  const long long ystride_v = (long long)(R + 1) * ldy;
  double2* o = out + m * out_mstride + (long long)r * (R + 1) + s;
  double2 phi = make_double2(0.0, 0.0), zeta = phi, delta = phi;
  if (s >= r) {
    const double2* Ym = Y + m * y_mstride + (long long)r * ldy;
    const double* eps_r = P.eps + (size_t)r * P.ldk;
    if (nonlin) {
      const double2 h0 = hshift(Ym + 4 * ystride_v, eps_r, r, s);
      const double2 h1 = hshift(Ym + 5 * ystride_v, eps_r, r, s);
      const double2 h2 = hshift(Ym + 6 * ystride_v, eps_r, r, s);
      const double2 p0 = Ym[s], p1 = Ym[ystride_v + s], p2 = Ym[2 * ystride_v + s];
      const double2 ke = Ym[3 * ystride_v + s];
      const double lam = lam_of(s, radius);
      phi = make_double2(p0.x + h0.x, p0.y + h0.y);
      zeta = make_double2(p1.x + h1.x, p1.y + h1.y);
      delta = make_double2(p2.x + h2.x - lam * ke.x, p2.y + h2.y - lam * ke.y);
    } else {
      zeta = Ym[s];
      delta = Ym[ystride_v + s];
    }
  }
  o[0] = phi;
  o[plane] = zeta;
  o[2 * plane] = delta;
}

__global__ void finalize_divcurl_kernel(PlanDev P, const double2* Y, long long y_mstride, int ldy,
                                        double2* div, double2* curl, int nmembers) {
  pdl_wait();
  pdl_trigger();
  const int R = P.R;
  const long long plane = (long long)(R + 1) * (R + 1);
  const long long total = (long long)nmembers * plane;
  const long long ystride_v = (long long)(R + 1) * ldy;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int m = (int)(idx / plane);
    const int rs = (int)(idx - m * plane);
    const int r = rs / (R + 1), s = rs - r * (R + 1);
    double2 d = make_double2(0.0, 0.0), c = d;
    if (s >= r) {
      const double2* Ym = Y + m * y_mstride + (long long)r * ldy;
      const double* eps_r = P.eps + (size_t)r * P.ldk;
      const double2 hd = hshift(Ym + ystride_v, eps_r, r, s);
      const double2 hc = hshift(Ym + 3 * ystride_v, eps_r, r, s);
      const double2 pd = Ym[s], pc = Ym[2 * ystride_v + s];
      d = make_double2(pd.x + hd.x, pd.y + hd.y);
      c = make_double2(pc.x + hc.x, pc.y + hc.y);
    }
    div[m * plane + rs] = d;
    curl[m * plane + rs] = c;
  }
}

// state layout: [m][3][R+1][R+1] complex, fields (phi', zeta, delta)
// Grid (s blocks, R + 1 rows, states).
__global__ void eval_fi_kernel(int R, ModelConsts c, const double2* x, double2* out,
                               long long nmat, RowFilter rf) {
  pdl_wait();
  pdl_trigger();
  const int s = blockIdx.x * blockDim.x + threadIdx.x, r = blockIdx.y;
  const long long m = blockIdx.z;
  if (s > R || r % rf.mod != rf.rank) return;
  (void)nmat;
  const long long plane = (long long)(R + 1) * (R + 1);
  const long long rs = (long long)r * (R + 1) + s;
  const double lam = lam_of(s, c.radius);
  const double nl = c.nu * lam;
  const double2* xm = x + m * 3 * plane + rs;
  double2* om = out + m * 3 * plane + rs;
  const double2 z0 = make_double2(0.0, 0.0);
  // s < r: structurally zero input (spharm.py:6-10), not read
  const bool up = s >= r;
  const double2 ph = up ? xm[0] : z0, ze = up ? xm[plane] : z0, de = up ? xm[2 * plane] : z0;
  om[0] = make_double2(-c.phi_bar * de.x + nl * ph.x, -c.phi_bar * de.y + nl * ph.y);
  om[plane] = make_double2(nl * ze.x, nl * ze.y);
  om[2 * plane] = make_double2(-lam * ph.x + nl * de.x, -lam * ph.y + nl * de.y);
}

__global__ void solve_kernel(int R, ModelConsts c, double beta, const double2* b, double2* out,
                             long long nmat, RowFilter rf) {
  pdl_wait();
  pdl_trigger();
  const long long plane = (long long)(R + 1) * (R + 1);
  const long long total = nmat * plane;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long m = idx / plane;
    const int rs = (int)(idx - m * plane);
    const int s = rs % (R + 1);
    if ((rs / (R + 1)) % rf.mod != rf.rank) continue;
    const double lam = lam_of(s, c.radius);
    const double d = 1.0 - beta * c.nu * lam;
    const double det = d * d - beta * beta * lam * c.phi_bar;
    const double id = 1.0 / det;
    const double bp = beta * c.phi_bar, bl = beta * lam;
    const double2* bm = b + m * 3 * plane + rs;
    double2* om = out + m * 3 * plane + rs;
    const double2 ph = bm[0], ze = bm[plane], de = bm[2 * plane];
    om[0] = make_double2((d * ph.x - bp * de.x) * id, (d * ph.y - bp * de.y) * id);
    om[plane] = make_double2(ze.x / d, ze.y / d);
    om[2 * plane] = make_double2((d * de.x - bl * ph.x) * id, (d * de.y - bl * ph.y) * id);
  }
}

__global__ void combine_kernel(CombineArgs a, long long count) {
  pdl_wait();
  pdl_trigger();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    double acc = 0.0;
    if (a.n > 0) acc = a.w[0] * a.x[0][i];
    for (int k = 1; k < a.n; ++k) acc = fma(a.w[k], a.x[k][i], acc);
    a.out[i] = acc;
  }
}

__global__ void laplacian_kernel(const double2* in, double2* out, int R, long long nmat,
                                 double radius, int inverse) {
  pdl_wait();
  pdl_trigger();
  const long long n = nmat * (R + 1) * (R + 1);
  const double a2 = radius * radius;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
       idx += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(idx % (R + 1));
    // lambda_s = -s (s + 1) / a^2 with the reference's rounding (spharm.py:307-310):
    // the product of two small integers is exact, one correctly rounded division
    const double lam = __ddiv_rn(-(double)s * ((double)s + 1.0), a2);
    const double2 v = in[idx];
    double2 o;
    if (!inverse) {
      o = make_double2(__dmul_rn(v.x, lam), __dmul_rn(v.y, lam));
    } else if (s == 0) {
      o = make_double2(0.0, 0.0);     // the singular s = 0 mode is gauged to zero
    } else {
      // numpy divides complex by real as Smith's complex division with a zero
      // imaginary part: one correctly rounded reciprocal, then two products
      const double scl = __drcp_rn(lam);
      o = make_double2(__dmul_rn(v.x, scl), __dmul_rn(v.y, scl));
    }
    out[idx] = o;
  }
}

__global__ void resize_kernel(const double2* in, int rin, double2* out, int rout, long long nmat,
                              RowFilter rf) {
  pdl_wait();
  pdl_trigger();
  const long long plane = (long long)(rout + 1) * (rout + 1);
  const long long total = nmat * plane;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long m = idx / plane;
    const int rs = (int)(idx - m * plane);
    const int r = rs / (rout + 1), s = rs - r * (rout + 1);
    if (r % rf.mod != rf.rank) continue;
    double2 v = make_double2(0.0, 0.0);
    if (r <= rin && s <= rin && s >= r) v = in[m * (long long)(rin + 1) * (rin + 1) + (long long)r * (rin + 1) + s];
    out[idx] = v;
  }
}

// Host -> device upload of spectral matrices reading only the s >= r triangle
// from page-locked host memory over PCIe (zero-copy); the lower triangle of the
// device copy is zero-filled locally.  kUp independent loads per thread keep
// enough PCIe read requests in flight to cover the round trip.
constexpr int kUp = 4;
__global__ void __launch_bounds__(256) upload_triangle_kernel(const double2* __restrict__ host,
                                                              double2* __restrict__ out, int R,
                                                              long long total) {
  pdl_wait();
  pdl_trigger();
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long base = blockIdx.x * (long long)blockDim.x + threadIdx.x; base < total;
       base += stride * kUp) {
    double2 v[kUp];
#pragma unroll
    for (int u = 0; u < kUp; ++u) {
      const long long i = base + u * stride;
      v[u] = make_double2(0.0, 0.0);
      if (i < total) {
        const int rs = (int)(i % ((long long)(R + 1) * (R + 1)));
        const int r = rs / (R + 1), s = rs - r * (R + 1);
        if (s >= r) v[u] = host[i];
      }
    }
#pragma unroll
    for (int u = 0; u < kUp; ++u) {
      const long long i = base + u * stride;
      if (i < total) out[i] = v[u];
    }
  }
}

// Device -> host download into page-locked memory by zero-copy stores: the
// s >= r triangle always, the (zero) lower triangle only when write_lower.
__global__ void __launch_bounds__(256) download_triangle_kernel(const double2* __restrict__ dev,
                                                                double2* __restrict__ host, int R,
                                                                long long total, int write_lower) {
  pdl_wait();
  pdl_trigger();
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long base = blockIdx.x * (long long)blockDim.x + threadIdx.x; base < total;
       base += stride * kUp) {
    double2 v[kUp];
    bool up[kUp];
#pragma unroll
    for (int u = 0; u < kUp; ++u) {
      const long long i = base + u * stride;
      up[u] = false;
      v[u] = make_double2(0.0, 0.0);
      if (i < total) {
        const int rs = (int)(i % ((long long)(R + 1) * (R + 1)));
        const int r = rs / (R + 1), s = rs - r * (R + 1);
        up[u] = s >= r;
        if (up[u]) v[u] = dev[i];
      }
    }
#pragma unroll
    for (int u = 0; u < kUp; ++u) {
      const long long i = base + u * stride;
      if (i < total && (up[u] || write_lower)) host[i] = v[u];
    }
  }
}

// Grid (s blocks, r_out + 1 rows, nout * nmat): one row (m, r) of one output
// per y/z coordinate, degrees s across x -- no per-element division.
__global__ void __launch_bounds__(256) spec_combine_multi_kernel(MultiCombineArgs a, int nmat,
                                                                 RowFilter rf) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.y;
  if (r % rf.mod != rf.rank) return;
  const int o = blockIdx.z / nmat, m = blockIdx.z - o * nmat;
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  const int ro = a.rout;
  if (r > a.ext[o] || s > a.ext[o]) return;
  double2 acc = make_double2(0.0, 0.0);
  // s < r is structurally zero in every spectral state (spharm.py:6-10): no reads
  if (s >= r)
  for (int k = a.off[o]; k < a.off[o + 1]; ++k) {
    const int ri = a.rin[k];
    if (r <= ri && s <= ri) {
      const double2 v = a.x[k][((size_t)m * (ri + 1) + r) * (ri + 1) + s];
      acc.x = fma(a.w[k], v.x, acc.x);
      acc.y = fma(a.w[k], v.y, acc.y);
    }
  }
  a.out[o][((size_t)m * (ro + 1) + r) * (ro + 1) + s] = acc;
}

__global__ void spec_combine_kernel(SpecCombineArgs a, long long nmat, RowFilter rf) {
  pdl_wait();
  pdl_trigger();
  const int ro = a.rout;
  const long long plane = (long long)(ro + 1) * (ro + 1);
  const long long total = nmat * plane;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long m = idx / plane;
    const int rs = (int)(idx - m * plane);
    const int r = rs / (ro + 1), s = rs - r * (ro + 1);
    if (r % rf.mod != rf.rank) continue;
    double2 acc = make_double2(0.0, 0.0);
    if (s >= r)   // s < r: structurally zero, no reads
    for (int k = 0; k < a.n; ++k) {
      const int ri = a.rin[k];
      if (r <= ri && s <= ri) {
        const double2 v = a.x[k][m * (long long)(ri + 1) * (ri + 1) + (long long)r * (ri + 1) + s];
        acc.x = fma(a.w[k], v.x, acc.x);
        acc.y = fma(a.w[k], v.y, acc.y);
      }
    }
    a.out[idx] = acc;
  }
}

// b = sum_k w_k x_k -> theta = (I - beta F_I)^-1 b -> fi = L_G(theta).
// Grid (s blocks, R + 1 rows, states): one row per y/z coordinate.
__global__ void sweep_node_kernel(int R, ModelConsts c, double beta, SpecCombineArgs a,
                                  double2* theta, double2* fi, long long nstates, RowFilter rf) {
  pdl_wait();
  pdl_trigger();
  const int s = blockIdx.x * blockDim.x + threadIdx.x, r = blockIdx.y;
  const long long m = blockIdx.z;
  if (s > R || r % rf.mod != rf.rank) return;
  (void)nstates;
  const long long plane = (long long)(R + 1) * (R + 1);
  const long long o = m * 3 * plane + (long long)r * (R + 1) + s;
  if (s < r) {
    // structurally zero coefficients (spharm.py:6-10): zeros out, no term reads
    const double2 z = make_double2(0.0, 0.0);
    theta[o] = z; theta[o + plane] = z; theta[o + 2 * plane] = z;
    fi[o] = z; fi[o + plane] = z; fi[o + 2 * plane] = z;
    return;
  }
  double2 b[3];
#pragma unroll
  for (int f = 0; f < 3; ++f) b[f] = make_double2(0.0, 0.0);
  for (int k = 0; k < a.n; ++k) {
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      const double2 v = a.x[k][o + f * plane];
      b[f].x = fma(a.w[k], v.x, b[f].x);
      b[f].y = fma(a.w[k], v.y, b[f].y);
    }
  }
  const double lam = lam_of(s, c.radius);
  const double d = 1.0 - beta * c.nu * lam;
  const double det = d * d - beta * beta * lam * c.phi_bar;
  const double id = 1.0 / det;
  const double bp = beta * c.phi_bar, bl = beta * lam;
  const double2 ph = make_double2((d * b[0].x - bp * b[2].x) * id, (d * b[0].y - bp * b[2].y) * id);
  const double2 ze = make_double2(b[1].x / d, b[1].y / d);
  const double2 de = make_double2((d * b[2].x - bl * b[0].x) * id, (d * b[2].y - bl * b[0].y) * id);
  theta[o] = ph;
  theta[o + plane] = ze;
  theta[o + 2 * plane] = de;
  const double nl = c.nu * lam;
  fi[o] = make_double2(-c.phi_bar * de.x + nl * ph.x, -c.phi_bar * de.y + nl * ph.y);
  fi[o + plane] = make_double2(nl * ze.x, nl * ze.y);
  fi[o + 2 * plane] = make_double2(-lam * ph.x + nl * de.x, -lam * ph.y + nl * de.y);
}

// Threads per row block of the (s, r, matrix) grids: the row length rounded up to a
// warp (<= 256), so a 171- or 86-entry row is one 192- or 96-thread block instead of two
// blocks with a third of their threads idle.
int row_threads(int row) { return row >= 256 ? 256 : ((row + 31) / 32) * 32; }

int grid_for(long long n, int threads) {
  long long b = (n + threads - 1) / threads;
  if (b > 148 * 16) b = 148 * 16;
  if (b < 1) b = 1;
  return (int)b;
}

}  // namespace

int launch_finalize_swe(const PlanDev& P, const double2* Y, long long y_mstride, int ldy,
                        double2* out, long long out_mstride, bool nonlin, double radius,
                        int nmembers, cudaStream_t st, RowFilter rf) {
  if (nmembers <= 0) return kOk;
  const int tx = row_threads(P.R + 1);
  const dim3 grid((P.R + 1 + tx - 1) / tx, P.R + 1, nmembers);
  StageScope sc("finalize_swe", st);
  SW_CUDA(launch_pdl(finalize_swe_kernel, grid, dim3(tx), 0, st, P, Y, y_mstride, ldy, out, out_mstride, nonlin ? 1 : 0, radius, nmembers, rf));
  SW_LAUNCH_CHECK();
  return kOk;
}

int launch_finalize_divcurl(const PlanDev& P, const double2* Y, long long y_mstride, int ldy,
                            double2* div, double2* curl, int nmembers, cudaStream_t st) {
  const long long n = (long long)nmembers * (P.R + 1) * (P.R + 1);
  StageScope sc("finalize_divcurl", st);
  SW_CUDA(launch_pdl(finalize_divcurl_kernel, dim3(grid_for(n, 256)), dim3(256), 0, st, P, Y, y_mstride, ldy, div, curl, nmembers));
  SW_LAUNCH_CHECK();
  return kOk;
}

int launch_eval_fi(int R, const ModelConsts& c, const double2* x, double2* out, long long nmat,
                   cudaStream_t st) {
  if (nmat <= 0) return kOk;
  const int tx = row_threads(R + 1);
  const dim3 grid((R + 1 + tx - 1) / tx, R + 1, (unsigned)nmat);
  StageScope sc("eval_fi", st);
  SW_CUDA(launch_pdl(eval_fi_kernel, grid, dim3(tx), 0, st, R, c, x, out, nmat, current_row_filter()));
  SW_LAUNCH_CHECK();
  return kOk;
}

int launch_solve(int R, const ModelConsts& c, double beta, const double2* b, double2* out,
                 long long nmat, cudaStream_t st) {
  const long long n = nmat * (R + 1) * (R + 1);
  StageScope sc("solve_implicit", st);
  SW_CUDA(launch_pdl(solve_kernel, dim3(grid_for(n, 256)), dim3(256), 0, st, R, c, beta, b, out, nmat, current_row_filter()));
  SW_LAUNCH_CHECK();
  return kOk;
}

int launch_combine(const CombineArgs& a, long long count, cudaStream_t st) {
  StageScope sc("combine", st);
  SW_CUDA(launch_pdl(combine_kernel, dim3(grid_for(count, 256)), dim3(256), 0, st, a, count));
  SW_LAUNCH_CHECK();
  return kOk;
}

int launch_spec_combine_multi(const MultiCombineArgs& a, long long nmat, cudaStream_t st) {
  if (a.nout <= 0 || nmat <= 0) return kOk;
  const int row = a.rout + 1;
  // the grid covers the largest output extent, not the array size: an in-place
  // interpolation into fine arrays only touches the coarse (r, s) square (config 4:
  // the 6-output interpolation launch ran 197k CTAs of which 3/4 of the threads
  // returned at once, 146 us at 2.6 TB/s)
  int ext = 0;
  for (int o = 0; o < a.nout; ++o) ext = std::max(ext, std::min(a.ext[o], a.rout) + 1);
  const int threads = ext >= 256 ? 256 : ((ext + 31) / 32) * 32;
  // gridDim.z = nout x matrices <= 65535: larger batches go in matrix chunks,
  // each launch with its inputs / outputs advanced to the chunk's first matrix
  const long long per = std::max(1LL, 65535LL / a.nout);
  StageScope sc("spec_combine", st);
  for (long long m0 = 0; m0 < nmat; m0 += per) {
    const int nm = (int)std::min(per, nmat - m0);
    MultiCombineArgs c = a;
    for (int k = 0; k < a.off[a.nout]; ++k)
      c.x[k] = a.x[k] + (size_t)m0 * (a.rin[k] + 1) * (a.rin[k] + 1);
    for (int o = 0; o < a.nout; ++o) c.out[o] = a.out[o] + (size_t)m0 * row * row;
    SW_CUDA(launch_pdl(spec_combine_multi_kernel,
                       dim3((ext + threads - 1) / threads, ext, (unsigned)(a.nout * nm)),
                       dim3(threads), 0, st, c, nm, current_row_filter()));
    SW_LAUNCH_CHECK();
  }
  return kOk;
}

int launch_spec_combine(const SpecCombineArgs& a, long long nmat, cudaStream_t st) {
  if ((long long)nmat <= 65535) {   // one output of the division-free multi kernel
    MultiCombineArgs m{};
    for (int k = 0; k < a.n; ++k) { m.x[k] = a.x[k]; m.w[k] = a.w[k]; m.rin[k] = a.rin[k]; }
    m.off[0] = 0;
    m.off[1] = a.n;
    m.out[0] = a.out;
    m.ext[0] = a.rout;
    m.nout = 1;
    m.rout = a.rout;
    return launch_spec_combine_multi(m, nmat, st);
  }
  const long long n = nmat * (a.rout + 1) * (a.rout + 1);
  StageScope sc("spec_combine", st);
  SW_CUDA(launch_pdl(spec_combine_kernel, dim3(grid_for(n, 256)), dim3(256), 0, st, a, nmat, current_row_filter()));
  SW_LAUNCH_CHECK();
  return kOk;
}

int launch_sweep_node(int R, const ModelConsts& c, double beta, const SpecCombineArgs& a,
                      double2* theta, double2* fi, long long nstates, cudaStream_t st) {
  if (nstates <= 0) return kOk;
  const int tx = row_threads(R + 1);
  const dim3 grid((R + 1 + tx - 1) / tx, R + 1, (unsigned)nstates);
  StageScope sc("sweep_node", st);
  SW_CUDA(launch_pdl(sweep_node_kernel, grid, dim3(tx), 0, st, R, c, beta, a, theta, fi, nstates, current_row_filter()));
  SW_LAUNCH_CHECK();
  return kOk;
}

int launch_laplacian(const double2* in, double2* out, int R, long long nmat, double radius,
                     int inverse, cudaStream_t st) {
  const long long n = nmat * (R + 1) * (R + 1);
  if (n == 0) return kOk;
  StageScope sc("laplacian", st);
  SW_CUDA(launch_pdl(laplacian_kernel, dim3(grid_for(n, 256)), dim3(256), 0, st, in, out, R, nmat,
                     radius, inverse));
  SW_LAUNCH_CHECK();
  return kOk;
}

int launch_resize(const double2* in, int rin, double2* out, int rout, long long nmat,
                  cudaStream_t st) {
  const long long n = nmat * (rout + 1) * (rout + 1);
  StageScope sc("resize", st);
  SW_CUDA(launch_pdl(resize_kernel, dim3(grid_for(n, 256)), dim3(256), 0, st, in, rin, out, rout, nmat, current_row_filter()));
  SW_LAUNCH_CHECK();
  return kOk;
}

int launch_upload_triangle(const double2* host, double2* out, int R, long long nmat,
                           cudaStream_t st) {
  const long long n = nmat * (R + 1) * (R + 1);
  StageScope sc("upload", st);
  // PCIe needs ~(bandwidth x round trip) ~ 100-200 KB of reads in flight; 32
  // CTAs (512 KB potential) keep the link busy while holding fewer memory-system
  // slots against the transforms running on other streams (8 CTAs: link-bound,
  // 64+: the concurrent transforms slow down).
  static const int cap = std::max(1, env_int("SWSDC_UPLOAD_CTAS", 32));
  const long long want = (n + 256LL * kUp - 1) / (256LL * kUp);
  const int blocks = (int)std::min<long long>(want, cap);
  SW_CUDA(launch_pdl(upload_triangle_kernel, dim3(blocks), dim3(256), 0, st, host, out, R, n));
  SW_LAUNCH_CHECK();
  return kOk;
}

__global__ void zero_lower_kernel(double2* out, int R, long long nmat) {
  pdl_wait();
  pdl_trigger();
  const long long total = nmat * (R + 1) * (R + 1);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int rs = (int)(i % ((long long)(R + 1) * (R + 1)));
    const int r = rs / (R + 1), s = rs - r * (R + 1);
    if (s < r) out[i] = make_double2(0.0, 0.0);
  }
}

// dst = src over n doubles; *bad = 1 if any value is not finite (*bad is
// cleared by the caller first): the graph stepper's state copy and per-step
// finiteness check (harness.py:257) in one pass.
// m-sharding exchange packing (distributed.py): blocks b of a [A][rows][cols][C]
// double array -- rows row0_b + k row_step_b (k < nrows_b), columns
// [col0_b, col1_b) -- gathered into (scatter = 0) or scattered from
// (scatter = 1) one contiguous buffer, block after block in order
// [b][A][k][col][C].  One launch replaces P strided copies per exchange.
__global__ void __launch_bounds__(256) exchange_blocks_kernel(ExchangeBlocks e, double* arr,
                                                               double* buf, int scatter) {
  pdl_wait();
  pdl_trigger();
  const long long total = e.off[e.nb];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    int b = 0;
    while (i >= e.off[b + 1]) ++b;
    long long rem = i - e.off[b];
    const int ncol = e.col1[b] - e.col0[b];
    const int c = (int)(rem % e.C);
    rem /= e.C;
    const int col = e.col0[b] + (int)(rem % ncol);
    rem /= ncol;
    const int k = (int)(rem % e.nrows[b]);
    const long long a = rem / e.nrows[b];
    const long long row = e.row0[b] + (long long)k * e.row_step[b];
    double* x = arr + ((a * e.rows + row) * e.cols + col) * e.C + c;
    if (scatter) *x = buf[i];
    else buf[i] = *x;
  }
}

__global__ void __launch_bounds__(256) copy_finite_kernel(const double* __restrict__ src,
                                                          double* __restrict__ dst, long long n,
                                                          int* bad) {
  pdl_wait();
  pdl_trigger();
  bool ok = true;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double v = src[i];
    dst[i] = v;
    ok = ok && isfinite(v);
  }
  if (!__all_sync(0xffffffffu, ok) && (threadIdx.x & 31) == 0) atomicExch(bad, 1);
}

int launch_exchange_blocks(const ExchangeBlocks& e, double* arr, double* buf, int scatter,
                           cudaStream_t st) {
  const long long n = e.off[e.nb];
  if (n == 0) return kOk;
  StageScope sc("exchange_pack", st);
  SW_CUDA(launch_pdl(exchange_blocks_kernel, dim3(grid_for(n, 256)), dim3(256), 0, st, e, arr, buf,
                     scatter));
  SW_LAUNCH_CHECK();
  return kOk;
}

int launch_copy_finite(const double* src, double* dst, long long n, int* bad, cudaStream_t st) {
  SW_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
  if (n <= 0) return kOk;
  StageScope sc("copy_finite", st);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long want = (n + 255) / 256;
  const int blocks = (int)std::min<long long>(want, 4LL * sms);
  SW_CUDA(launch_pdl(copy_finite_kernel, dim3(blocks), dim3(256), 0, st, src, dst, n, bad));
  SW_LAUNCH_CHECK();
  return kOk;
}

int launch_zero_lower(double2* out, int R, long long nmat, cudaStream_t st) {
  const long long n = nmat * (R + 1) * (R + 1);
  StageScope sc("zero_lower", st);
  SW_CUDA(launch_pdl(zero_lower_kernel, dim3(grid_for(n, 256)), dim3(256), 0, st, out, R, nmat));
  SW_LAUNCH_CHECK();
  return kOk;
}

int launch_download_triangle(const double2* dev, double2* host, int R, long long nmat,
                             int write_lower, cudaStream_t st) {
  const long long n = nmat * (R + 1) * (R + 1);
  StageScope sc("download", st);
  static const int cap = std::max(1, env_int("SWSDC_UPLOAD_CTAS", 32));
  const long long want = (n + 256LL * kUp - 1) / (256LL * kUp);
  const int blocks = (int)std::min<long long>(want, cap);
  SW_CUDA(launch_pdl(download_triangle_kernel, dim3(blocks), dim3(256), 0, st, dev, host, R, n, write_lower));
  SW_LAUNCH_CHECK();
  return kOk;
}

}  // namespace swsdc
