// TMA-fed streaming products over M (fp64), csrc/tma_prod.cu.
//
// Both write split-K partials in the layouts the fixed-order k_sum_partials of
// csrc/anls.cu finishes:
//   row product  part[chunk][row][p] = sum_{j in chunk} M[row][j] B[j][p]   (B: cols x K)
//   col product  part[split][col][p] = sum_{i in split} M[i][col] B[i][p]   (B: rows x K)
// Return NMFB_EUNSUPPORTED when the shape / alignment does not fit (the caller then
// uses the register-direct kernels); *nparts receives the number of partials.
#pragma once
#include "common.cuh"

// column chunk of the TMA row product (B chunk resident in shared memory); the same
// partial count as the register-direct k_rowprod_mma (MMA_CW), so work lengths agree
constexpr int TMA_RP_CW = 512;

bool tma_prod_enabled();
int tma_rowprod_f64(const double* A, long rows, long cols, const double* B, int K, double* work,
                    long work_len, long* nparts, cudaStream_t st);
int tma_colprod_f64(const double* A, long rows, long cols, const double* B, int K, double* work,
                    long work_len, long* nparts, cudaStream_t st);
// number of row splits tma_colprod_f64 uses (work >= splits * cols * K)
long tma_colprod_splits(long rows, long cols);
// ONE pass over M for outR = M B1 (row partials left in work[0 : nch rows K] for the
// caller's fixed-order k_sum_partials, nch = ceil(cols / TMA_RP_CW)) and outC = M^T B2
// (finished here).  K in 5..16.
long tma_dualprod_work_len(long rows, long cols, long k);
int tma_dualprod_f64(const double* A, long rows, long cols, const double* B1, const double* B2,
                     int K, double* outR, double* outC, double* work, long work_len,
                     cudaStream_t st);
// fp32 M (c5): TMA-fed FP64 tensor-core column product; *nparts = 2 x the row splits
int tma_colprod_f32(const float* A, long rows, long cols, const double* B, int K, double* work,
                    long work_len, long* nparts, cudaStream_t st);
