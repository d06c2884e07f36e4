// ORACLE (test infrastructure only): thread control of the CPU restatement.
//
// The reference's solve path is single-threaded.  The oracle may run its loops over independent
// rows, blocks, columns and aggregates on several threads: every such unit is computed with exactly
// the sequential code's operation order and written to its own output slot, so every result is
// bitwise independent of the thread count (tests/test_oracle_parallel.py checks setup, applies and
// GMRES at 1 vs N threads).  Reductions (GMRES dot products and norms, the AMG aggregation BFS)
// always stay sequential.  Default: 1 thread.
#pragma once

#include <algorithm>
#include <exception>
#include <mutex>
#include <vector>

#include "fpo.hpp"

namespace fpo {

int threads();
void set_threads(int n);

// First exception thrown inside a parallel loop, rethrown after it (an exception must not leave an
// OpenMP region).  Records the one from the lowest index, so the error is the sequential code's.
class LoopError {
 public:
  void capture(long idx) {
    std::lock_guard<std::mutex> g(m_);
    if (!err_ || idx < idx_) err_ = std::current_exception(), idx_ = idx;
  }
  void rethrow() const {
    if (err_) std::rethrow_exception(err_);
  }

 private:
  std::mutex m_;
  std::exception_ptr err_;
  long idx_ = 0;
};

// Rows built in parallel chunks, each row with the sequential code (fn appends row i's entries),
// stitched in row order: the output does not depend on the schedule.
template <class Scratch, class MakeScratch, class RowFn>
CsrMatrix build_rows(int n_rows, int n_cols, MakeScratch make_scratch, RowFn fn) {
  constexpr int kChunk = 4096;
  const int nch = (n_rows + kChunk - 1) / kChunk;
  std::vector<std::vector<int>> cols(static_cast<size_t>(nch));
  std::vector<std::vector<double>> vals(static_cast<size_t>(nch));
  CsrMatrix C(n_rows, n_cols);
  LoopError err;
#pragma omp parallel num_threads(threads())
  {
    Scratch sc = make_scratch();
#pragma omp for schedule(dynamic)
    for (int c = 0; c < nch; ++c) {
      try {
        for (int i = c * kChunk; i < std::min(n_rows, (c + 1) * kChunk); ++i) {
          fn(i, sc, cols[c], vals[c]);
          C.row_offsets[size_t(i) + 1] = int64_t(cols[c].size());  // chunk-local for now
        }
      } catch (...) {
        err.capture(c);
      }
    }
  }
  err.rethrow();
  std::vector<int64_t> base(static_cast<size_t>(nch) + 1, 0);
  for (int c = 0; c < nch; ++c) base[c + 1] = base[c] + int64_t(cols[c].size());
  C.col_indices.resize(size_t(base[nch]));
  C.values.resize(size_t(base[nch]));
#pragma omp parallel for num_threads(threads()) schedule(dynamic)
  for (int c = 0; c < nch; ++c) {
    for (int i = c * kChunk; i < std::min(n_rows, (c + 1) * kChunk); ++i) C.row_offsets[size_t(i) + 1] += base[c];
    std::copy(cols[c].begin(), cols[c].end(), C.col_indices.begin() + base[c]);
    std::copy(vals[c].begin(), vals[c].end(), C.values.begin() + base[c]);
    std::vector<int>().swap(cols[c]);
    std::vector<double>().swap(vals[c]);
  }
  return C;
}

}  // namespace fpo
