// tcgen05 (tf32 x 3 split) streaming products over an fp32 M, csrc/tc_prod.cu.
#pragma once
#include "common.cuh"

constexpr int TC_RP_CW = 512;  // column chunk of the row product (= MMA_CW partial count)

bool tc_prod_enabled();
// part[chunk][row][p] = sum_{j in chunk} M[row][j] B[j][p] (fp64 partials, *nparts chunks)
int tc_rowprod_f32(const float* A, long rows, long cols, const double* B, int K, double* work,
                   long work_len, long* nparts, cudaStream_t st);
// part[split][col][p] = sum_{i in split} M[i][col] X[i][p] (fp64 partials, *nparts splits)
int tc_colprod_f32(const float* A, long rows, long cols, const double* X, int K, double* work,
                   long work_len, long* nparts, cudaStream_t st);
