// dict_internal.h -- the dictionary object shared by dict.cu (Phi_D, subspace basis) and llr.cu
// (the LLR outer step uses the basis).  Internal; the public handle is mrf_dict.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <vector>

#include "../../include/mrfnufft.h"

struct mrf_dict_s {
  int K = 0, L = 0, P = 0, device = 0;
  int NP = 0;                    // GEMM rows (2 K padded to 256)
  float2* atoms = nullptr;       // [K][L] complex64 (the exact rescoring)
  double* dn2 = nullptr;         // [K] ||d_k||^2 (float64)
  float* lut = nullptr;          // [K][P]
  // certified filter of Phi_D (match.cuh): Rf <= 64 orthonormal rows phi of the dictionary's
  // leading right singular vectors, the atoms' coefficients a_k = phi d_k packed as fp16
  // [a_hi | a_hi | a_lo] rows, the filter weights (m_k / ||d_k||)^2 and the error bound beta
  int Rf = 0;
  float2* phi = nullptr;         // [64][L] (rows past Rf zero)
  float2* phiT = nullptr;        // [L][64]
  __half* dpf = nullptr;         // [NP][KF]
  float* w2f = nullptr;          // [NP / 2] (m_k / ||d_k||)^2 (normalised correlation, reading 21)
  float* w2f2 = nullptr;         // [NP / 2] (m_k / ||d_k||^2)^2 (Eq. 5 as printed, MRF_MATCH_NORM2)
  double dmin = 0.0;             // smallest non-zero atom norm (the printed form's band)
  CUtensorMap tmdf;
  double beta = 0.0;             // |rho~_k - rho_k| <= beta for every atom and voxel (the GEMM filter)
  double2* a64 = nullptr;        // [K][64] a_k = phi d_k (float64; the rescoring's second level)
  double* beta2 = nullptr;       // [K] |rho^_k - rho_k| bound of the float64 coefficient score
  double beta_res = 0.0, beta_a1 = 0.0;   // max ||r_k|| / ||d_k||, max ||a_k||_1 / ||d_k|| (diagnostics)
  // per-voxel workspaces (grown on demand)
  __half* xp = nullptr;          // [vcap][KF] packed filter coefficients
  float* xs = nullptr;           // [vcap] per-voxel scale
  double* xnorm = nullptr;       // [vcap] ||x_v||
  double2* u64 = nullptr;        // [vcap][64] u = phi x (float64 totals of fp32 chunks)
  unsigned long long* best = nullptr;   // [vcap] packed (score, ~atom) maxima of the filter pass
  float* thr = nullptr;          // [vcap] certified-band threshold
  int* ncand = nullptr;          // [vcap]
  int* cand = nullptr;           // [vcap][kCand]
  int* ov = nullptr;             // [vcap] voxels rescored against every atom
  int* nov = nullptr;            // [1]
  void* part_best = nullptr;     // [vcap][16] per-part bests of the full scan (match.cuh PartBest)
  long long vcap = 0;
  float2* xT = nullptr;          // [vtcap][L] voxel-major frames (frame-domain match)
  long long vtcap = 0;
  bool prof = false;             // CUDA events around the tensor-core GEMMs (mrf_dict_profile)
  std::vector<cudaEvent_t> ev;   // pairs
  size_t ev_used = 0;
  double fro2 = 0.0;             // ||D||_F^2 (float64, at creation)
  int rank = 0;                  // subspace basis (mrf_dict_basis): r rows of length L
  unsigned basis_gen = 0;        // process-wide generation of the basis (mrf_dict_basis)
  float2* basis = nullptr;       // device [rank][L]
  std::vector<float2> basis_h;   // host copy
  // the match in basis coordinates (mrf_dict_match_coef, x = sum_i w_i d_i): Gd = d d^H
  // [rank][rank] and Dc [K][rank] = <d_i, d_k> (float64), and the r-dimensional filter
  double2* Gd = nullptr;
  double2* Dc = nullptr;
  __half* dpc = nullptr;         // [NP][KFC] packed [Dc_hi | Dc_hi | Dc_lo] / m'_k rows (the coefficient filter)
  float* w2c = nullptr;          // [NP / 2] (m'_k / ||d_k||)^2
  float* w2c2 = nullptr;         // [NP / 2] (m'_k / ||d_k||^2)^2
  CUtensorMap tmdc;
  double beta_c = 0.0;           // the coefficient filter's bound on |rho~_k - rho_k|
  // last match: voxels rescored against every atom (diagnostics)
  int last_overflow = 0;
};
