// Launch interfaces of the Legendre stage (legendre.cu).
#pragma once
#include "common.cuh"

namespace swsdc {

enum SynMode : int { kSynPlain = 0, kSynUV = 1, kSynSWE = 2 };

// Output layout of synthesis: eo[b][r][jh][2] double2 = (E, O), the even- and
// odd-degree partial sums at the north latitude of pair jh.
struct SynArgs {
  const double2* src;      // plain: B fields; UV: psi; SWE: state (phi, zeta, delta)
  const double2* src2;     // UV: chi
  long long src_fstride;   // complex elements between fields of src
  int src_R;               // truncation of the input arrays (<= plan R; coarser inputs are zero-padded)
  int smax;                // highest degree synthesised (R, or R+1 when H is folded onto P)
  double radius;           // SWE: planet radius (psi = zeta / lambda, U/a, V/a)
  double2* eo;             // output
  long long src_mstride;   // complex elements between members (blockIdx.y)
  long long eo_mstride;    // double2 elements between members
  int nmembers;            // independent states / field groups in one launch
  const int2* pairs;       // optional row pairs (r1, r2; r2 < 0: single row); default {p, R-p}
  int npairs;
  int nJB;                 // set by the launcher
};

// Input of analysis: the weighted north+south (S) and north-south (D) Fourier
// combinations of nv vectors in the fragment-native XLayout (common.cuh);
// x points at the vector group being analysed.
struct AnaArgs {
  const double* x;
  XLayout xl;
  int nv;                  // number of vectors in this group (<= 16)
  double2* out;            // out[v * out_vstride + r * out_rstride + s]
  long long out_vstride;
  long long out_rstride;
  int smax;                // highest degree written (R, or R+1 for the H shift)
  int zero_fill;           // also write zeros for s < r
  const int4* work;        // (r, first chunk c, checkpoint index ck_off[r] + c, 0) list,
                           // one CTA (ana_warps_per_cta chunks) each
  long long out_mstride;   // complex elements between members (blockIdx.y)
  int nmembers;
  int short_tiles;         // run half-empty last chunks without their upper m-tile
};

int build_checkpoints(const PlanDev& P, const double* a_tab, const double* b_tab,
                      const double* sect_fac, double2* ckpt, cudaStream_t st);
int launch_synthesis(const PlanDev& P, const SynArgs& a, int B, int mode, cudaStream_t st);
int launch_analysis(const PlanDev& P, const AnaArgs& a, int nwork, int lsplit, cudaStream_t st);
int ana_warps_per_cta();
// chunks per CTA of the register analysis kernel for a latitude split (1..4)
int ana_chunks_per_cta(int lsplit);
int ana_ctas_per_sm(int nv, int lsplit, bool tab);
// Whether the analysis of nt n-tiles x mp members per CTA streams A from P.ptab.
bool ana_table_fed(const PlanDev& P, int nt, int mp);
// Fragment-native Pbar table for the table-fed analysis (see build_ptab in legendre.cu):
// nck chunks x jh4 4-latitude blocks x 128 doubles; ptab must be zero-initialised.
// syn = 1: the synthesis-order table (P.stab, see syn_dmma_kernel): per (chunk, 32-latitude
// block) 8 k-steps x 128 doubles.
int build_ptab(const PlanDev& P, const double* a_tab, const double* b_tab, const double* sect_fac,
               double* ptab, cudaStream_t st, int syn = 0);
int launch_synthesis_dmma(const PlanDev& P, const SynArgs& a, int nf, cudaStream_t st);
constexpr int kAnaSplits = 4;
bool ana_uses_tma(int nv);
bool ana_dfma_enabled();   // SWSDC_ANA_DFMA comparison kernel selected
// Ensemble analysis two members per CTA (a.nmembers = member pairs, nv <= 8
// vectors each, members m and m + 1 adjacent at a.xl.mstride / a.out_mstride).
bool ana_pairs_ok(int nv, int nmembers);
int launch_analysis_pairs(const PlanDev& P, const AnaArgs& a, int nwork, int lsplit, cudaStream_t st);

}  // namespace swsdc
