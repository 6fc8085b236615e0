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
  int KD = 0, NP = 0;            // fp16 row length (2 L padded to 64), GEMM rows (2 K padded to 256)
  __half* dp = nullptr;          // [NP][KD] atom rows (re/im rotated, scaled by 1 / m_k)
  float* w2 = nullptr;           // [NP / 2] (m_k / ||d_k||)^2, 0 for padding
  float* n2inv = nullptr;        // [K] 1 / ||d_k||^2 (0 for a zero atom)
  float2* atoms = nullptr;       // [K][L] complex64 (for the exact pd)
  float* lut = nullptr;          // [K][P]
  __half* xp = nullptr;          // workspace [vcap][KD]
  float* xs = nullptr;           // [vcap] per-voxel scale
  unsigned long long* best = nullptr;   // [vcap] packed (score, ~atom) running maxima
  long long vcap = 0;
  CUtensorMap tmd;
  bool prof = false;             // CUDA events around the tensor-core GEMM (mrf_dict_profile)
  std::vector<cudaEvent_t> ev;   // pairs
  size_t ev_used = 0;
  double fro2 = 0.0;             // ||D||_F^2 (float64, at creation)
  int rank = 0;                  // subspace basis (mrf_dict_basis): r rows of length L
  unsigned basis_gen = 0;        // incremented by every mrf_dict_basis
  float2* basis = nullptr;       // device [rank][L]
  std::vector<float2> basis_h;   // host copy
  // the dictionary in basis coordinates, Dc = D d^dagger [K][rank] (mrf_dict_match_coef): packed
  // fp16 rows like dp (row length 64 >= 2 rank) and w2c = (m'_k / ||d_k||)^2 with the FULL atom
  // norms, so that scores and pd equal those of the frame-domain match for x in span(d)
  __half* dpc = nullptr;         // [NP][64]
  float* w2c = nullptr;          // [NP / 2]
  float2* Dc = nullptr;          // [K][rank]
  CUtensorMap tmdc;
};
