// TEST INFRASTRUCTURE ONLY — see oracle.hpp.  Dense and banded Cholesky used by
// the oracle in place of Eigen's LLT / SimplicialLLT (src/dd.cpp:66-76,
// src/sg.cpp:218-225).
#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <mutex>
#include <thread>

#include "oracle.hpp"

namespace oracle {

namespace {
inline double dot(const double* a, const double* b, Index n) {
  double s = 0.0;
#pragma omp simd reduction(+ : s)
  for (Index k = 0; k < n; ++k) s += a[k] * b[k];
  return s;
}
inline void axpy(double alpha, const double* x, double* y, Index n) {
#pragma omp simd
  for (Index k = 0; k < n; ++k) y[k] -= alpha * x[k];
}
}  // namespace

// Row-oriented Cholesky-Crout; Eigen LLT semantics: fails on pivot <= 0.
bool Llt::compute(const Dense& m) {
  n = m.rows;
  l.assign(static_cast<size_t>(n) * n, 0.0);
  ok = true;
  for (Index i = 0; i < n; ++i) {
    double* li = &l[static_cast<size_t>(i) * n];
    for (Index j = 0; j <= i; ++j) {
      const double* lj = &l[static_cast<size_t>(j) * n];
      const double s = m(i, j) - dot(li, lj, j);
      if (j < i) {
        li[j] = s / lj[j];
      } else {
        if (!(s > 0.0)) {
          ok = false;
          return false;
        }
        li[i] = std::sqrt(s);
      }
    }
  }
  return true;
}

void Llt::solve_in_place(double* b) const {
  for (Index i = 0; i < n; ++i) {
    const double* li = &l[static_cast<size_t>(i) * n];
    b[i] = (b[i] - dot(li, b, i)) / li[i];
  }
  for (Index i = n - 1; i >= 0; --i) {
    const double* li = &l[static_cast<size_t>(i) * n];
    b[i] /= li[i];
    axpy(b[i], li, b, i);
  }
}

// src/dd.cpp:66-76
Llt llt_regularized(Dense m) {
  Llt llt;
  if (llt.compute(m) || m.rows == 0) {
    llt.ok = true;
    return llt;
  }
  double trace = 0.0;
  for (Index i = 0; i < m.rows; ++i) trace += m(i, i);
  const double shift = 1e-10 * trace / m.rows;
  for (Index i = 0; i < m.rows; ++i) m(i, i) += shift;
  if (!llt.compute(m)) throw std::runtime_error("llt_regularized: factorization failed after regularization");
  return llt;
}

bool BandLlt::compute(Index n_, Index bw_, const std::function<void(Index, double*)>& fill_row) {
  n = n_;
  bw = bw_;
  const Index w = bw + 1;
  l.assign(static_cast<size_t>(n) * w, 0.0);
  for (Index i = 0; i < n; ++i) {
    double* li = &l[static_cast<size_t>(i) * w];  // li[j - i + bw]
    fill_row(i, li);                              // A(i, i-bw .. i) into li
    const Index j0 = std::max<Index>(0, i - bw);
    for (Index j = j0; j <= i; ++j) {
      const double* lj = &l[static_cast<size_t>(j) * w];
      const Index k0 = std::max<Index>(j0, j - bw);  // common range [k0, j)
      const double s = li[j - i + bw] - dot(li + (k0 - i + bw), lj + (k0 - j + bw), j - k0);
      if (j < i) {
        li[j - i + bw] = s / lj[bw];
      } else {
        if (!(s > 0.0)) return false;
        li[bw] = std::sqrt(s);
      }
    }
  }
  return true;
}

void BandLlt::solve_in_place(double* b) const {
  const Index w = bw + 1;
  for (Index i = 0; i < n; ++i) {
    const double* li = &l[static_cast<size_t>(i) * w];
    const Index k0 = std::max<Index>(0, i - bw);
    b[i] = (b[i] - dot(li + (k0 - i + bw), b + k0, i - k0)) / li[bw];
  }
  for (Index i = n - 1; i >= 0; --i) {
    const double* li = &l[static_cast<size_t>(i) * w];
    const Index k0 = std::max<Index>(0, i - bw);
    b[i] /= li[bw];
    axpy(b[i], li + (k0 - i + bw), b + k0, i - k0);
  }
}

// b is row-major n x nrhs; rows before `first` are known to be zero.
void BandLlt::solve_many(double* b, Index nrhs) const {
  const Index w = bw + 1;
  Index first = 0;
  while (first < n) {
    bool nz = false;
    for (Index c = 0; c < nrhs && !nz; ++c) nz = b[static_cast<size_t>(first) * nrhs + c] != 0.0;
    if (nz) break;
    ++first;
  }
  for (Index i = first; i < n; ++i) {
    const double* li = &l[static_cast<size_t>(i) * w];
    double* bi = b + static_cast<size_t>(i) * nrhs;
    for (Index k = std::max<Index>(first, i - bw); k < i; ++k)
      axpy(li[k - i + bw], b + static_cast<size_t>(k) * nrhs, bi, nrhs);
    const double inv = 1.0 / li[bw];
#pragma omp simd
    for (Index c = 0; c < nrhs; ++c) bi[c] *= inv;
  }
  for (Index i = n - 1; i >= 0; --i) {
    const double* li = &l[static_cast<size_t>(i) * w];
    double* bi = b + static_cast<size_t>(i) * nrhs;
    const double inv = 1.0 / li[bw];
#pragma omp simd
    for (Index c = 0; c < nrhs; ++c) bi[c] *= inv;
    for (Index k = std::max<Index>(0, i - bw); k < i; ++k)
      axpy(li[k - i + bw], bi, b + static_cast<size_t>(k) * nrhs, nrhs);
  }
}

// include/sgwave/parallel.hpp:20-43: strided assignment, first exception rethrown.
void parallel_for(int n, int n_threads, const std::function<void(int)>& fn) {
  if (n <= 0) return;
  n_threads = std::max(1, std::min(n_threads, n));
  if (n_threads == 1) {
    for (int i = 0; i < n; ++i) fn(i);
    return;
  }
  std::exception_ptr error;
  std::mutex mu;
  std::vector<std::thread> workers;
  for (int t = 0; t < n_threads; ++t)
    workers.emplace_back([&, t] {
      try {
        for (int i = t; i < n; i += n_threads) fn(i);
      } catch (...) {
        std::lock_guard<std::mutex> lock(mu);
        if (!error) error = std::current_exception();
      }
    });
  for (auto& w : workers) w.join();
  if (error) std::rethrow_exception(error);
}

}  // namespace oracle
