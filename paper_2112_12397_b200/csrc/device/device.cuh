// Device-side data layout of the B200 solve path.
//
// Every sparse operator is stored "sliced by 32 rows" (SELL-32): within a slice,
// the k-th stored entry of each of the 32 rows is contiguous, so one warp step
// is one fully coalesced 256-byte load per stream.  One thread owns one output
// row and accumulates it left to right in the reference's CSR order
// (csr.cpp:109-119), which makes every SpMV bitwise equal to the CPU oracle
// while streaming HBM at full width.
//
//  * Sell  — scalar CSR rows (C1, Q1, C2, H, Q2, T, coarse A_l, P_l, R_l = P_l^T).
//  * Bsr3  — 3x3-block rows (A and the inner-AMG fine operator S~ / S1): per
//            slice and block slot k, 9 x 32 doubles laid out [li][j][lane], read
//            by three warps (li = 0,1,2), plus one int block column per slot.
//            8.44 B per scalar nonzero instead of CSR's 12 B.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace fpd {

// layout constants shared by the builders (formats.cu) and the kernels (kernels.cuh)
constexpr int kSlice = 32;                        // rows (block rows, nodes) per SELL slice
constexpr int kPipeRows = 32, kPipeW = 32;        // windowed pipeline: rows per slice, entries per window row
constexpr int kPipeCtasPerSm = 2;                 // two resident pipelines per SM (registers capped at 128)

struct SellView {
  int n_rows = 0;
  const long long* slice_off = nullptr;  // slot index of (slice, k=0, lane=0)
  const int* row_len = nullptr;
  const int* cols = nullptr;
  const double* vals = nullptr;
  // optional (sell_kernel only): rows sorted by length inside windows of kSellWindow rows before
  // slicing, slot -> row (-1 = padding); null: slot = row
  int n_slots = 0;
  const int* rows = nullptr;
};
constexpr int kSellWindow = 2048;

// Node-blocked rows (the finest prolongation P_1 with a 3x3-block fine level): the three
// scalar rows of a node share one column pattern, so a slot holds one column index and
// three values.  SELL-32 over nodes: slot (slice s, k, lane) at q = slice_off[s] + 32 k + lane;
// its column at cols[q], its values at vals[3 (slice_off[s] + 32 k) + 32 d + lane], d = 0..2.
// Nodes are sorted by length inside windows of kBp3Window nodes before they are sliced (slot ->
// node in `node`, -1 = padding), so the 32 nodes of a slice have nearly one length and a slice
// stores (and streams) almost no padding.
constexpr int kBp3Window = 2048;
struct Bp3View {
  int n_nodes = 0;
  const long long* slice_off = nullptr;
  const int* node_len = nullptr;
  const int* cols = nullptr;
  const double* vals = nullptr;
  int n_slots = 0;            // 32 * slices
  const int* node = nullptr;  // n_slots: the node of slot (slice, lane)
};

struct CsrView {  // plain CSR, 64-bit offsets (warp-per-row kernel)
  int n_rows = 0;
  const long long* rp = nullptr;
  const int* ci = nullptr;
  const double* v = nullptr;
  const int* row_map = nullptr;  // optional (csr_warp_kernel): compute only rows row_map[0 .. n_rows)
  // optional (csr_warp_kernel): groups of consecutive rows share one column list (the coarse dofs of
  // an aggregate); entry k of row r has its value at v[k] and its column at ci[cp[r] + (k - rp[r])]
  const long long* cp = nullptr;
};

// Quad-per-row layout for the strided32 row sums of operators with many rows (AMG level 1 and its
// restriction at the large configs).  Rows are sorted by length inside windows of kSrtWindow rows
// and cut into slices of 8 (slot -> row in `row`, -1 = padding); a warp takes a slice, four lanes
// per row: lane (rl, q) owns the partials 8 q .. 8 q + 7 of row rl and, in round t, the row's entries
// 32 t + 8 q + u (u = 0..7).  Values: vals[slice_off[slice] + ((8 t + u) * 8 + rl) * 4 + q], so the
// warp's u-th load of a round is one 256-byte line; columns: CSR lists shared by runs of
// equal-pattern rows (share_columns), entry k of row r at ci[cp[r] + k].
constexpr int kSrtWindow = 2048, kSrtRows = 8;
struct SrtView {
  int n_slices = 0;
  const int* row = nullptr;              // 8 per slice
  const long long* slice_off = nullptr;  // n_slices + 1; a slice holds 256 values per round
  const int* row_len = nullptr;
  const long long* cp = nullptr;
  const int* ci = nullptr;
  const double* vals = nullptr;
  const int* out_row = nullptr;  // optional (row-subset copy): local row r is the operator's row out_row[r]
};

// Windowed slices for the ordered long-row pipeline (csr_pipe_kernel): rows
// grouped 32 to a slice (sorted by length inside chunks of 4096 rows to cut
// padding), each slice stored as windows of 32 x 32 slots [window][row][lane]
// holding entries w*32 + lane of each row in CSR order (padding: 0.0, column 0).
struct PipeView {
  int n_slices = 0;
  const long long* woff = nullptr;  // n_slices + 1: first window of each slice
  const int* row = nullptr;         // 32 per slice: original row index (-1 = padding)
  const int* len = nullptr;         // 32 per slice: row length
  const double* v = nullptr;
  const int* ci = nullptr;
  const int* cta_slice = nullptr;   // persistent CTAs: CTA b owns slices [cta_slice[b], cta_slice[b+1])
};

struct Bsr3View {
  int n_brows = 0;
  const long long* slice_off = nullptr;  // block-slot index of (slice, k=0, lane=0)
  const int* brow_len = nullptr;
  const int* bcols = nullptr;            // one per block slot
  const double* vals = nullptr;          // 9 per block slot, [li][j][lane] inside each (slice,k) group
  float l2_keep = 0.f;                   // > 0: fraction of lines loaded evict-last (bsr3_kernel<.., true>)
  const int* brow_map = nullptr;         // optional: block row b of this (row-subset) matrix is global row brow_map[b]
};

struct BandView {
  int n = 0, kl = 0, ku = 0, n_blocks = 0;
  const int* block_start = nullptr;
  const double* Lc = nullptr;    // n * kl, column j multipliers L(j+1+r, j)
  const double* diag = nullptr;  // D (spd) or U diagonal (general)
  const double* Lr = nullptr;    // spd: n * kl, L(j, j-1-r)
  const double* Uc = nullptr;    // general: n * ku, U(j-1-r, j)
  const int* piv = nullptr;      // general: absolute row swapped with j at step j
  int spd = 1;
  int pivoted = 1;               // general: 0 when the LU took no row swaps
};

// factor_solve = inverse: explicit inverse of every fracture block, row-major,
// block b at off[b] (rows of all blocks stacked in factor order).
struct DinvView {
  const int* block_start = nullptr;
  const long long* off = nullptr;
  const double* v = nullptr;
};

// factor_solve = panel: per block, panels of p rows with the dense H, G, K, F of the
// oracle's BandFactor::build_panels (fpo.hpp), stacked per block at off[blk].
constexpr int kPanelMax = 256;  // largest panel (bandwidth) the device path takes
struct PanelView {
  int n_blocks = 0;
  const int* block_start = nullptr;
  const int* p = nullptr;           // panel size per block
  const long long* off = nullptr;   // per block: offset of its panel matrices
  const double* m = nullptr;
  const double* diag = nullptr;     // spd: D (z = y / D between the sweeps); null for general
  int m_max = 0;                    // largest block (rows)
  int p_max_panels = 0;             // most panels of a block: each warp keeps its own rows of x per panel
  double* z = nullptr;              // n doubles of scratch: z = y / D (or y), written by the forward chain
  const int* order = nullptr;       // cluster c solves block order[c]: longest chains first
};

struct DenseLUView {  // coarse-level full-pivot LU, column-major n x n
  int n = 0, rank = 0;
  const double* lu = nullptr;
  const int* prow = nullptr;
  const int* pcol = nullptr;
};

// Arnoldi step status, written by the device into mapped host memory
struct GmresStatus {
  double est, hnext, wnorm_pre;
  int happy, nonfinite, reorth, m;
};

// Programmatic dependent launch: every kernel of the apply first waits for its
// predecessor grid to complete (and its writes to be visible), then lets the
// next grid in the stream launch.  The successor's CTAs are scheduled into this
// grid's tail instead of after a full drain + launch gap.  Without a programmatic
// dependency (ordinary launches) both instructions return immediately.
__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---------------------------------------------------------------- buffers
void cuda_check(cudaError_t e, const char* what);

template <class T>
class DevBuf {
 public:
  DevBuf() = default;
  explicit DevBuf(size_t n) { alloc(n); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr, o.n_ = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p_ = o.p_, n_ = o.n_;
      o.p_ = nullptr, o.n_ = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t n) {
    release();
    n_ = n;
    if (n) cuda_check(cudaMalloc(&p_, n * sizeof(T)), "cudaMalloc");
  }
  void upload(const T* h, size_t n) {
    alloc(n);
    if (n) cuda_check(cudaMemcpy(p_, h, n * sizeof(T), cudaMemcpyHostToDevice), "cudaMemcpy H2D");
  }
  void upload(const std::vector<T>& h) { upload(h.data(), h.size()); }
  void zero() {
    if (n_) cuda_check(cudaMemset(p_, 0, n_ * sizeof(T)), "cudaMemset");
  }
  T* get() const { return p_; }
  size_t size() const { return n_; }
  size_t bytes() const { return n_ * sizeof(T); }

 private:
  void release() {
    if (p_) cudaFree(p_);
    p_ = nullptr;
    n_ = 0;
  }
  T* p_ = nullptr;
  size_t n_ = 0;
};

}  // namespace fpd
