// Interface systems from caller-built LocalSchur data and the generic PCG
// (generic.cu).
#pragma once
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <deque>
#include <functional>
#include <memory>
#include <vector>

#include "solver.cuh"

namespace sgw {

using DevOp = std::function<void(const double* x_dev, double* y_dev)>;

// src/pcg.cpp:7-50 on device vectors (x0 = 0); returns the iteration count
int pcg_generic(cublasHandle_t blas, cudaStream_t st, long long n, const DevOp& op, const DevOp& pre,
                const double* b_dev, double* x_dev, double tol, int max_iter, bool* converged,
                std::vector<double>* hist);

void spd_inverse_inplace(cusolverDnHandle_t sol, cudaStream_t st, double* A, int n);

class GenericSchur {
 public:
  struct LocalInput {  // include/sgwave/dd.hpp:50-62 (host arrays, copied)
    int n = 0, nr = 0, nc = 0;
    const double* S = nullptr;  // n x n column-major
    const long long* gmap = nullptr;
    const double* weights = nullptr;
    const int *r_idx = nullptr, *c_idx = nullptr;
    const long long* corner_gmap = nullptr;
  };
  GenericSchur(long long n_global, long long n_corner, const std::vector<LocalInput>& locals);
  ~GenericSchur();
  GenericSchur(const GenericSchur&) = delete;
  GenericSchur& operator=(const GenericSchur&) = delete;
  void matvec(const double* x_dev, double* y_dev);
  void apply_nn2(const double* r_dev, double* z_dev);
  const std::vector<double>& coarse_operator() const { return fcc_; }  // F_cc (n_corner^2, column-major)
  long long n_global() const { return n_global_; }
  cudaStream_t stream() const { return st_; }
  cublasHandle_t blas() const { return blas_; }

 private:
  struct Local {
    int n = 0, nr = 0, nc = 0;
    DBuf<double> S, w, Srr_inv, Src;
    DBuf<long long> gmap, cgmap;
    DBuf<int> ridx, cidx;
  };
  long long n_global_, n_corner_;
  int maxn_ = 0;
  std::vector<std::unique_ptr<Local>> locals_;
  std::deque<DBuf<double>> tloc_;
  std::vector<double> fcc_;
  DBuf<double> Finv_, xl_, yl_, t_, d_, uc_;
  cudaStream_t st_ = nullptr;
  cublasHandle_t blas_ = nullptr;
  cusolverDnHandle_t sol_ = nullptr;
};

}  // namespace sgw
