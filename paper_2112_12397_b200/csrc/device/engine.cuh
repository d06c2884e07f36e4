// Device engine: uploaded operators, the inner AMG V-cycle, the t-p-u / t-u-p /
// t-u-p* block-triangular applies and the restarted GMRES driver.  Host code in
// this file only enqueues work; everything on the solve path runs on the GPU.
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <deque>
#include <memory>
#include <vector>

#include "../host/setup.hpp"
#include "device.cuh"

namespace fpd {

// Algorithmic HBM bytes of the kernels an operation enqueues:
// each stored matrix once per use, each vector once per read or write.
struct Ledger {
  double bytes = 0.0;
  int launches = 0;
  double wasted = 0.0;  // bytes a launch streams beyond its algorithmic bytes (explicit block inverses)
  void add(double b) { bytes += b, ++launches; }
  void waste(double b) { wasted += b; }
};

struct DSell {
  int n_rows = 0, n_cols = 0, n_slices = 0;
  long long slots = 0;
  int64_t nnz = 0;
  DevBuf<long long> off;
  DevBuf<int> len, cols, rows;  // rows: slot -> row of the length-sorted variant (sell_from(.., sorted))
  DevBuf<double> vals;
  SellView view() const {
    return {n_rows, off.get(), len.get(), cols.get(), vals.get(), int(rows.size()), rows.size() ? rows.get() : nullptr};
  }
  double matrix_bytes() const { return 12.0 * double(nnz) + 4.0 * (n_rows + 1) + 4.0 * double(rows.size()); }  // CSR-equivalent
};

struct DBsr3 {
  int n_brows = 0, n_slices = 0;
  long long slots = 0;
  int64_t nblocks = 0;
  DevBuf<long long> off;
  DevBuf<int> len, bcols;
  DevBuf<double> vals;
  float l2_keep = 0.f;  // finest AMG operator: fraction kept L2-resident across sweeps
  DevBuf<int> brow_map;  // row-subset matrices: global block row of each block row
  Bsr3View view() const { return {n_brows, off.get(), len.get(), bcols.get(), vals.get(), l2_keep, brow_map.get()}; }
  double matrix_bytes() const { return 76.0 * double(nblocks) + 4.0 * (n_brows + 1); }
};

DSell make_sell(const fpb::Csr& A);

struct DBp3 {  // node-blocked rows (Bp3View)
  int n_nodes = 0;
  int64_t nnz = 0, slots = 0;
  DevBuf<long long> off;
  DevBuf<int> len, cols, node;
  DevBuf<double> vals;
  Bp3View view() const {
    return {n_nodes, off.get(), len.get(), cols.get(), vals.get(), int(node.size()), node.get()};
  }
  // format bytes: one column index per node entry + three values
  double matrix_bytes() const { return 28.0 * double(nnz) / 3.0 + 4.0 * (n_nodes + 1) + 4.0 * double(node.size()); }
};
// empty (n_nodes = 0) unless the three rows of every node share one column pattern
DBp3 make_bp3(const fpb::Csr& A);
// A square, n % 3 == 0; brows: only these block rows (in order; their global indices go to brow_map)
DBsr3 make_bsr3(const fpb::Csr& A, const std::vector<int>* brows = nullptr);


// Plain CSR on the device, consumed one warp per row (csr_warp_kernel).
struct DCsr {
  int n_rows = 0, n_cols = 0;
  int64_t nnz = 0;
  DevBuf<long long> rp;
  DevBuf<int> ci;
  DevBuf<double> v;
  // shared column lists (formats.cu share_columns): ci holds nci < nnz indices, cp the per-row offset
  DevBuf<long long> cp;
  int64_t nci = 0;
  CsrView view() const {
    CsrView V{n_rows, rp.get(), ci.get(), v.get()};
    V.cp = cp.size() ? cp.get() : nullptr;
    return V;
  }
  double index_bytes_per_entry() const { return cp.size() && nnz > 0 ? 4.0 * double(nci) / double(nnz) : 4.0; }
  double row_bytes() const { return cp.size() ? 16.0 : 8.0; }  // offsets read per row
  double matrix_bytes() const { return (8.0 + index_bytes_per_entry()) * double(nnz) + row_bytes() * (n_rows + 1); }
};

}  // namespace fpd
namespace fpb {
struct DeviceMatrix {  // setup.hpp: a device-resident level operator
  fpd::DCsr m;
};
}  // namespace fpb
namespace fpd {

struct DSrt {  // quad-per-row strided32 layout (SrtView)
  int n_rows = 0;
  int64_t nnz = 0, nci = 0, slots = 0;
  DevBuf<int> row, len, ci, out_row;  // out_row: set for a row-subset copy (srt_subset_from)
  DevBuf<long long> off, cp;
  DevBuf<double> vals;
  SrtView view() const {
    return {int(row.size() / kSrtRows), row.get(), off.get(), len.get(), cp.get(), ci.get(), vals.get(),
            out_row.size() ? out_row.get() : nullptr};
  }
  // values once, the shared column lists once, per row: slot -> row, length, list offset (+ slice offsets)
  double matrix_bytes() const { return 8.0 * double(nnz) + 4.0 * double(nci) + 17.0 * n_rows; }
};
// the layout of A (same entries, same order per row); shares column lists where rows allow
DSrt srt_from(const DCsr& A, cudaStream_t s);
// the same layout for the rows rows[0 .. m) of A only (A may carry shared column lists); local row t
// computes A's row rows[t]
DSrt srt_subset_from(const DCsr& A, const std::vector<int>& rows, cudaStream_t s);

struct DPipe {
  int n_rows = 0, n_slices = 0, n_ctas = 0;
  int64_t nnz = 0, slots = 0;
  DevBuf<long long> woff;
  DevBuf<int> row, len, ci, cta_slice;
  DevBuf<double> v;
  PipeView view() const {
    return {n_slices, woff.get(), row.get(), len.get(), v.get(), ci.get(), cta_slice.get()};
  }
  double matrix_bytes() const { return 12.0 * double(nnz) + 8.0 * n_rows; }
};
DPipe make_pipe(const fpb::Csr& A);

// A scalar sparse operator in the layout that streams best for its shape:
// SELL-32 (thread per row) for many short rows, warp-row CSR for few / long
// rows (coarse AMG levels, restrictions).  Both sum each row left to right.
struct DMat {
  bool warp = false;
  int slice_rows = 32;  // rows per CTA of the slice kernel (8 for few-row operators)
  bool pipe = false;     // warp && many rows: the windowed producer/consumer pipeline
  bool strided = false;  // row_sum = strided32 (extension): csr_warp_kernel / csr_slice_strided_kernel
  bool bp3 = false;      // node-blocked rows (finest prolongation): bp3_kernel
  DBp3 bp;
  bool srt = false;      // strided && many rows: quad-per-row srt_kernel for full launches (csr stays for row subsets)
  DSrt sr;
  int strided_rows = 4;  // rows per CTA of csr_slice_strided_kernel
  DSell sell;
  DCsr csr;
  DPipe pm;
  int n_rows() const { return bp3 ? 3 * bp.n_nodes : pipe ? pm.n_rows : warp ? csr.n_rows : sell.n_rows; }
  int64_t nnz() const { return bp3 ? bp.nnz : pipe ? pm.nnz : warp ? csr.nnz : sell.nnz; }
  double matrix_bytes() const {
    return bp3 ? bp.matrix_bytes() : srt ? sr.matrix_bytes() : pipe ? pm.matrix_bytes() : warp ? csr.matrix_bytes() : sell.matrix_bytes();
  }
};
// few_rows_parallel: operators with under 2048 rows take the row-parallel slice kernel even
// for short rows (a thread-per-row chain would be the whole kernel's latency)
DMat make_mat(const fpb::Csr& A, bool few_rows_parallel = false, bool strided = false);

// A host CSR borrowed for an upload (no copy): the reference's layout with 64-bit row offsets.
struct HostCsrView {
  int n_rows = 0, n_cols = 0;
  const int64_t* rp = nullptr;
  const int* ci = nullptr;
  const double* v = nullptr;
  int64_t nnz() const { return n_rows > 0 ? rp[n_rows] : 0; }
  static HostCsrView of(const fpb::Csr& A) { return {A.n_rows, A.n_cols, A.rp.data(), A.ci.data(), A.v.data()}; }
};
struct SystemView {  // BlockSystem (block.hpp:36-45) as borrowed views
  int n_u = 0, n_t = 0, n_p = 0;
  HostCsrView A, C1, Q1, C2, H, Q2, T, F_u;
  static SystemView of(const fpb::HostSystem& J) {
    return {J.n_u, J.n_t, J.n_p, HostCsrView::of(J.A), HostCsrView::of(J.C1), HostCsrView::of(J.Q1),
            HostCsrView::of(J.C2), HostCsrView::of(J.H), HostCsrView::of(J.Q2), HostCsrView::of(J.T),
            HostCsrView::of(J.F_u)};
  }
};

// ---- device-side layout builders (formats.cu): CSR in HBM -> the solve path's layouts
DCsr upload_csr(const HostCsrView& A);
inline DCsr upload_csr(const fpb::Csr& A) { return upload_csr(HostCsrView::of(A)); }
fpb::Csr download_csr(const DCsr& A);
// sorted: rows sorted by length inside windows before slicing (for sell_kernel launches only)
DSell sell_from(const DCsr& A, cudaStream_t s, bool sorted = false);
DBp3 bp3_from(const DCsr& A, cudaStream_t s);
DBsr3 bsr3_from(const DCsr& A, const std::vector<int>* brows, cudaStream_t s);
DPipe pipe_from(const DCsr& A, cudaStream_t s);
DCsr transpose_dev(const DCsr& A, cudaStream_t s);  // rows of A^T list the source rows ascending
DMat mat_from(DCsr&& A, bool few_rows_parallel, bool strided, cudaStream_t s);
bool sell_sorted();
// Rows with exactly their predecessor's columns share that row's list (ci shrinks, cp gives each
// row its list); returns false and leaves A as it is when under 1/8 of the indices would go.  The
// entries and their order per row do not change.
bool share_columns(DCsr& A, cudaStream_t s);

fpb::Csr host_copy(const HostCsrView& A);
DCsr add_dev(const DCsr& A, const DCsr& B, double alpha, double beta);  // alpha A + beta B (dsetup.cu)
// C = diag(row_scale) A B on the device, bitwise the host spgemm (spgemm.cu); row_scale may be null
DCsr spgemm_dev(const DCsr& A, const DCsr& B, const double* row_scale_dev);
// build_tpu / build_tup with the fine-size setup on the device (dsetup.cu); the AMG levels of the
// result stay device-resident (HostLevel::dA / dP)
fpb::HostPrecond build_precond_device(const SystemView& J, const fpb::HostSystem* Jh, int variant,
                                      const fpb::AmgOptions& opt, const std::vector<std::array<double, 3>>& coords);

}  // namespace fpd
namespace fpb {
struct FractureModel;
}
namespace fpd {

// The state-dependent blocks C2, H, T, F_u, Q2 assembled on the device from a fracture state
// (assembly.cu; assemble_fracture_blocks, assembly.cpp:229-406): the model (faces, edges, Dirichlet
// flags, constants) is uploaded once, run() rebuilds the blocks for every new state.
class DeviceFractureAssembly {
 public:
  explicit DeviceFractureAssembly(const fpb::FractureModel& m);
  ~DeviceFractureAssembly();
  void run(const char* region, const double* gap, const double* trac, const double* sdir, const double* pres);
  int n_u = 0, n_p = 0;
  DCsr C2, H, T, F_u, Q2;

 private:
  struct Model;
  std::unique_ptr<Model> model_;
};

class DeviceSystem {
 public:
  explicit DeviceSystem(const fpb::HostSystem& J);
  explicit DeviceSystem(const SystemView& J);
  ~DeviceSystem();
  DeviceSystem(const DeviceSystem&) = delete;
  DeviceSystem& operator=(const DeviceSystem&) = delete;
  int n_u = 0, n_t = 0, n_p = 0;
  // the t/p rows (jtp_kernel) run on a side stream, concurrently with the A rows (fork/join
  // through events; captured into the graphs as parallel branches)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int n() const { return n_u + n_t + n_p; }
  double st = 1.0, sp = 1.0;  // driver block scaling (driver.cpp:114-125)
  bool a_bsr3 = true;         // A as 3x3 blocks (n_u = 3 * nodes); SELL otherwise
  DBsr3 A;
  DSell A_sell;
  DSell C1, Q1, C2, H, Q2, T;
  DMat Q2m;  // Q2 for the preconditioner's s_p / t_p products (layout chosen by make_mat)
  // y = D J D x (D = blkdiag(I, st I, sp I)); st = sp = 1 gives J itself
  void enqueue_apply(const double* x, double* y, double st_, double sp_, cudaStream_t s, Ledger* L = nullptr) const;
  double bytes_apply() const;
  // a Newton step's new C2, H, T, Q2 (device CSR, e.g. DeviceFractureAssembly): layouts and the block
  // scaling rebuilt on the device; A, C1, Q1 unchanged
  void set_fracture_blocks(const DCsr& C2, const DCsr& H, const DCsr& T, const DCsr& Q2);
  double max_diag_A = 0.0;
};

struct DeviceLevel {
  bool bsr3 = false;
  DBsr3 Ab;
  DMat Am;
  DMat P, R;  // P: this level <- next coarser; R = P^T (level l+1 holds P_{l+1}, R_{l+1})
  DevBuf<double> d, b, x, xt, xt2, xt3, r;
  // Chebyshev smoother (extension): coefficients of this level and its direction vector
  double cheb_theta = 0.0;
  std::vector<double> cheb_c1, cheb_c2;
  DevBuf<double> cd;
  // multicolour Gauss-Seidel smoother (extension): the level operator as CSR, rows grouped by colour
  DCsr gs;
  DevBuf<int> color_rows;
  std::vector<int> color_off;
  int n = 0;
  double a_bytes() const { return bsr3 ? Ab.matrix_bytes() : Am.matrix_bytes(); }
};

class DeviceAmg {
 public:
  DeviceAmg(const fpb::HostAmg& h, bool fine_bsr3);
  int n_levels() const { return int(lv.size()); }
  int fine_n() const { return lv.empty() ? 0 : lv[0].n; }
  // x = amg_apply(r) (amg.cpp:293-305); if sub_from != null writes sub_from - x instead.
  // xhat, if given, already holds the first Jacobi sweep from zero, (omega r_i) / d_i, computed
  // by the kernel that produced r (it is used as scratch and overwritten).
  void enqueue_apply(const double* r, double* x, const double* sub_from, cudaStream_t s, Ledger* L = nullptr,
                     double* xhat = nullptr, bool sparse_rhs = false);
  // Sparse right-hand sides (t-u-p's second V-cycle: t_u2 = Q1 v_p is +0 off the rows Q1 touches):
  // block rows of level 0 whose residual can be nonzero, and rows of R_1 that can gather a nonzero;
  // every other row's sum is an exact +0, so those rows skip their loads (bitwise the full sweep).
  void set_sparse_rhs(const std::vector<unsigned char>& rhs_rows);
  // the levels' CSR in HBM while the upload cuts row subsets from them (borrowed from the device
  // setup or uploaded into own_), dropped by release_build_data
  std::vector<const DCsr*> src_A_, src_P_;
  std::deque<DCsr> own_;
  void release_build_data() {
    src_A_.clear(), src_P_.clear();
    own_.clear();
  }
  struct SpLevel {             // the sparse pass at one level (§10f)
    DBsr3 fine;                // level 0: the operator restricted to the block rows whose residual can be nonzero
    DevBuf<int> res_rows;      // level >= 1: those rows (warp-row kernel row list)
    int res_n = 0;
    double res_bytes = 0.0;
    DSrt res_srt;              // ... or their quad-per-row copy when the level's operator uses that layout
    DevBuf<int> r_rows;        // rows of R_{l+1} that can gather a nonzero
    int r_n = 0;
    double r_bytes = 0.0;
    DSrt r_srt;
    DevBuf<double> r, bnext;   // this level's residual and the next level's rhs: +0 off the active rows
  };
  std::vector<SpLevel> sp_lv;  // levels 0 .. sp_lv.size()-1 run the sparse pass
  bool sp_ready = false;
  std::vector<int> level_sizes() const;
  std::vector<DeviceLevel> lv;
  DevBuf<double> lu;
  DevBuf<int> prow, pcol;
  int coarse_n = 0, coarse_rank = 0;
  DevBuf<double> top_x, top_res, top_dx;
  fpb::AmgOptions opt;
  // when set, the finest level's Jacobi post-sweep of a V-cycle without sub_from (the bench's
  // roofline kernel) is bracketed by these two events, recorded into the captured graph
  cudaEvent_t probe_ev[2] = {nullptr, nullptr};
  // one V-cycle from level l (amg.cpp:151-177); public for the per-level profile
  void vcycle(int l, const double* b, double* x, const double* sub_from, double* xhat, cudaStream_t s, Ledger* L,
              bool sparse_rhs = false);

 private:
  void vcycle_chebyshev(int l, const double* b, double* x, const double* sub_from, cudaStream_t s, Ledger* L);
  void vcycle_mcgs(int l, const double* b, double* x, const double* sub_from, cudaStream_t s, Ledger* L);
};

class DevicePrecond {
 public:
  DevicePrecond(const DeviceSystem& sys, const fpb::HostPrecond& hp);
  int variant = 1;
  const DeviceSystem* sys;
  std::unique_ptr<DeviceAmg> amg;
  DevBuf<double> hlu;
  DevBuf<int> hpiv;
  BandView band{};
  DevBuf<int> band_start, band_piv;
  DevBuf<double> band_Lc, band_diag, band_Lr, band_Uc;
  int band_max_block = 0;
  // factor_solve = inverse: explicit block inverses streamed by dinv_kernel
  bool inverse = false;
  // factor_solve = panel: block-bidiagonal panels, panel_solve_kernel
  bool panel = false;
  PanelView pview{};
  DevBuf<int> pan_p, pan_order;
  DevBuf<long long> pan_off;
  DevBuf<double> pan_m, pan_z;
  size_t pan_smem = 0;
  double pan_bytes = 0;
  int pan_pmax = 0;
  DinvView dinv{};
  DevBuf<double> dinv_v;
  DevBuf<long long> dinv_off;
  double dinv_bytes = 0;
  double band_factor_bytes = 0;  // B_factor of SURVEY §8(d): 12 (nnz(L) + nnz(U)) + diagonal (+ pivots)
  DevBuf<double> tt, tu, tp, su, sp_, vp, tu2, vu2, xh;
  long inner_calls = 0;
  int inner_per_apply() const { return variant == 1 ? 2 : 1; }
  // y = D^-1 M D^-1 x with at = 1/st, ap = 1/sp (at = ap = 1: M itself)
  void enqueue_apply(const double* x, double* y, double at, double ap, cudaStream_t s, Ledger* L = nullptr);
  void enqueue_band(const double* rhs, double rs, double* out, double* out2, const double* sub, double os, int mode,
                    cudaStream_t s, Ledger* L);
};

constexpr int kOrthMgs = 0, kOrthCgs = 1;  // FP_ORTH_*
struct SolveOptions {
  int orth = kOrthMgs;
  bool probe = false;  // time the roofline kernel in every Arnoldi step (CUDA events in the graph)
  double tol = 1e-10;
  int restart = 50;
  int max_iter = 500;
  bool scaled = true;
};

struct SolveResult {
  int iterations = 0, restarts = 0, precond_applies = 0;
  bool converged = false, breakdown = false;
  double final_rel_residual = 0.0;
  std::vector<double> history;
  double device_seconds = 0.0;
  long long launches = 0;
  double probe_ms = 0.0;  // summed CUDA-event time of the probed kernel
  int probe_count = 0;
  int reorth_steps = 0;   // Arnoldi steps that ran the DGKS second pass
};

struct ProfileResult {
  double apply_ms = 0, apply_bytes = 0, japply_ms = 0, japply_bytes = 0;
  double fine_resid_ms = 0, fine_resid_bytes = 0, fine_post_ms = 0, fine_post_bytes = 0;
  double band_ms = 0, band_bytes = 0, coarse_ms = 0;
  double apply_wasted_bytes = 0;
  int apply_launches = 0;
  std::vector<double> vcycle_ms;  // graph of the V-cycle from level l down
};
ProfileResult profile_precond(const DeviceSystem& sys, DevicePrecond& pc, int reps, cudaStream_t s);

struct MgsArgs;   // gmres_kernels.cuh
struct CgsState;

// Restarted right-preconditioned GMRES on the device (gmres.cpp semantics per
// cycle + the GMRES(m) wrapper of SURVEY §8(a) G1).
class GmresSolver {
 public:
  GmresSolver(const DeviceSystem& sys, DevicePrecond& pc, int restart);
  ~GmresSolver();
  SolveResult solve(const double* b_dev, double* x_dev, const SolveOptions& o, cudaStream_t s);
  double apply_bytes = 0.0, japply_bytes = 0.0;  // algorithmic bytes of one precond / J apply
  int apply_launches = 0, japply_launches = 0;

 private:
  void build_graphs(double st, double sp, bool probe, cudaStream_t s);
  double norm_into(const double* a, const double* b, double* diff_out, double* dev_out, cudaStream_t s);
  const DeviceSystem& sys_;
  DevicePrecond& pc_;
  int restart_, ldr_;
  long long n_, ldv_;
  DevBuf<double> V_, z_, jout_, xtot_, r_, dx_, partial_, h_, cs_, sn_, g_, R_, y_, scal_;
  DevBuf<int> flag_;
  GmresStatus* status_h_ = nullptr;
  GmresStatus* status_d_ = nullptr;
  double* host_scalar_ = nullptr;
  double* host_scalar_d_ = nullptr;
  int mgs_grid_ = 0, red_grid_ = 0;
  int mgs_ept_ = 0;       // > 0: mgs_fast_kernel<E> (slices in registers / shared memory)
  int big_nblk_ = 0;      // classical GS for large n: tiles of the wide-kernel chain
  DevBuf<double> big_coef_;
  DevBuf<CgsState> big_state_;
  size_t mgs_smem_ = 0;
  void launch_mgs(MgsArgs& a, int orth, cudaStream_t s);
  // [0] the apply + J graph; with probe, [1] / [2] the same graph with a probe event pair
  // each, used by every kProbeEvery-th Arnoldi step (alternating)
  cudaGraphExec_t pj_exec_[3] = {nullptr, nullptr, nullptr}, j_exec_ = nullptr;
  static constexpr int kProbeEvery = 8;
  double graph_st_ = -1, graph_sp_ = -1;
  bool graph_probe_ = false;
  cudaEvent_t probe_ev_[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
};

}  // namespace fpd
