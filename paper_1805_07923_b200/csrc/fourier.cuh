// Launch interfaces of the longitude stage (fourier.cu).
#pragma once
#include "common.cuh"

namespace swsdc {

// (E, O) partial sums of nf fields -> grids [nf][I][J]
int launch_fourier_to_grid(const PlanDev& P, const double2* eo, long long eo_fstride, double* grid,
                           long long grid_fstride, int nf, cudaStream_t st, int jh_begin = 0,
                           int jh_end = -1);
// (E, O) partial sums of nf fields -> rings [nf][Jh][I] (double2 north, south),
// the grid layout of the split F_E path
int launch_fourier_to_rings(const PlanDev& P, const double2* eo, long long eo_fstride,
                            double2* rings, long long ring_fstride, int nf, cudaStream_t st,
                            int jh_begin = 0, int jh_end = -1);
// grids -> weighted (S, D) vectors in XLayout.  mode 0: plain (nf fields = nf
// vectors of one member); mode 1: div/curl (nf (U, V) pairs = nf members of 4 vectors)
int launch_grid_to_fourier(const PlanDev& P, int mode, const double* grid, const double* grid2,
                           long long grid_fstride, double* x, const XLayout& xl, int nf,
                           cudaStream_t st);
// fused eval_f_e grid stage for nmembers states
int launch_swe_grid(const PlanDev& P, bool nonlinear, const double2* eo, long long eo_mstride,
                    double* x, const XLayout& xl, int nmembers, double omega, double radius,
                    cudaStream_t st, int jh_begin = 0, int jh_end = -1);

// true when the fused grid kernel's 7 rings fit in shared memory
bool swe_grid_fits(const PlanDev& P);
bool swe_split_preferred(const PlanDev& P, long long pair_members);
bool fourier_reg_fft(const PlanDev& P);
int launch_swe_split_reg(const PlanDev& P, bool nonlinear, const double2* eo, long long eo_fstride,
                         double2* ring_ws, double* x, const XLayout& xl, int nmembers,
                         double omega, double radius, cudaStream_t st, int jh_begin, int jh_end);
// large-n_lon path: products + forward FFTs from 5 grids in HBM in the ring
// layout (double2 rings[m * gmember + q * gfield + jh * I + il], q = U/a, V/a,
// zeta, delta, phi'; strides in double2)
int launch_swe_products(const PlanDev& P, bool nonlinear, const double* grids, long long gfield,
                        long long gmember, const double2* eo, long long eo_fstride, double* x,
                        const XLayout& xl, int nmembers, double omega, double radius,
                        cudaStream_t st, int jh_begin = 0, int jh_end = -1);

}  // namespace swsdc
