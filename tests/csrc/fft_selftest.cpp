// CPU self-test of the shared-memory FFT index math (csrc/fft_core.cuh):
// forward DIF (digit-reversed output) and inverse DIT (digit-reversed input)
// against a naive O(n^2) DFT for every ring length the BASELINE configs use
// plus odd / prime lengths.  Built and run by tests/test_fft_core.py.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "../../paper_1805_07923_b200/csrc/fft_core.cuh"

int main(int argc, char** argv) {
  int sizes[] = {1, 2, 3, 4, 5, 6, 7, 8, 10, 12, 13, 14, 16, 22, 24, 25, 32, 33, 48, 50, 64, 96, 100, 125, 128, 143, 192, 256, 2048,
                 384, 512, 768, 1920, 3840};
  double worst = 0.0;
  for (int n : sizes) {
    std::vector<double2> tw(n), x(n), y(n), ref(n);
    for (int e = 0; e < n; ++e) {
      long double a = -2.0L * 3.14159265358979323846264338327950288L * e / n;
      tw[e].x = (double)cosl(a); tw[e].y = (double)sinl(a);
    }
    srand(n);
    for (int i = 0; i < n; ++i) { x[i].x = rand() / (double)RAND_MAX - 0.5; x[i].y = rand() / (double)RAND_MAX - 0.5; }
    for (int k = 0; k < n; ++k) {
      long double sr = 0, si = 0;
      for (int i = 0; i < n; ++i) {
        long double a = -2.0L * 3.14159265358979323846264338327950288L * (((long long)i * k) % n) / n;
        sr += x[i].x * cosl(a) - x[i].y * sinl(a);
        si += x[i].x * sinl(a) + x[i].y * cosl(a);
      }
      ref[k].x = (double)sr; ref[k].y = (double)si;
    }
    swfft::FftPlan p = swfft::make_fft_plan(n);
    // forward on a padded ring
    std::vector<double2> buf(swfft::padded_len(n));
    for (int i = 0; i < n; ++i) buf[swfft::pad_idx(i)] = x[i];
    swfft::fft_forward_dif_serial(buf.data(), p, tw.data());
    double err = 0;
    for (int k = 0; k < n; ++k) {
      int pos = swfft::pad_idx(swfft::digit_rev(p, k));
      err = fmax(err, fabs(buf[pos].x - ref[k].x) + fabs(buf[pos].y - ref[k].y));
    }
    // forward DIT (kernel path): digit-reversed input, natural output
    std::vector<double2> d(swfft::padded_len(n));
    for (int i = 0; i < n; ++i) d[swfft::pad_idx(swfft::digit_rev(p, i))] = x[i];
    swfft::fft_dit_serial<false>(d.data(), p, tw.data());
    for (int k = 0; k < n; ++k) {
      const double2 dk = d[swfft::pad_idx(k)];
      err = fmax(err, fabs(dk.x - ref[k].x) + fabs(dk.y - ref[k].y));
    }
    // inverse: place ref (spectrum) digit-reversed, run inverse, expect n * x
    std::vector<double2> z(swfft::padded_len(n));
    for (int k = 0; k < n; ++k) z[swfft::pad_idx(swfft::digit_rev(p, k))] = ref[k];
    swfft::fft_dit_serial<true>(z.data(), p, tw.data());
    double err2 = 0;
    for (int i = 0; i < n; ++i) {
      const double2 zi = z[swfft::pad_idx(i)];
      err2 = fmax(err2, fabs(zi.x / n - x[i].x) + fabs(zi.y / n - x[i].y));
    }
    printf("n=%5d stages=%d fwd_err=%.3e inv_err=%.3e\n", n, p.nstage, err, err2);
    worst = fmax(worst, fmax(err / sqrt((double)n), err2));
  }
  printf("WORST %.3e\n", worst);
  return worst < 1e-13 ? 0 : 1;
}
