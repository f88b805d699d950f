// Launch interfaces of the longitude stage (fourier.cu).
#pragma once
#include "common.cuh"

namespace swsdc {

// (E, O) partial sums of nf fields -> grids [nf][I][J]
int launch_fourier_to_grid(const PlanDev& P, const double2* eo, long long eo_fstride, double* grid,
                           long long grid_fstride, int nf, cudaStream_t st);
// grids -> weighted (S, D) vectors.  mode 0: plain (nf fields, 1 vector each);
// mode 1: div/curl (nf (U, V) pairs, 4 vectors each, x_fstride per pair)
int launch_grid_to_fourier(const PlanDev& P, int mode, const double* grid, const double* grid2,
                           long long grid_fstride, double2* x, long long x_fstride, int nf,
                           cudaStream_t st);
// fused eval_f_e grid stage for nmembers states
int launch_swe_grid(const PlanDev& P, bool nonlinear, const double2* eo, long long eo_mstride,
                    double2* x, long long x_mstride, int nmembers, double omega, double radius,
                    cudaStream_t st);

}  // namespace swsdc
