// Synthetic workload generator (see workload.hpp).  Mesh rules follow
// /root/reference/proj/core/src/mesh.cpp:51-224; assembly follows
// assembly.cpp:39-97 (element), 132-188 (elasticity + Dirichlet elimination),
// 190-216 (C1/Q1), 229-406 (C2, H, T, F_u, Q2).  Per-entry accumulation of the
// stiffness is deterministic (cells are colored by index parity and scattered
// color by color) but not the reference's cell order; this generator only feeds
// both the oracle and the GPU path with the same matrices.
#include "workload.hpp"

#include <omp.h>

#include <algorithm>
#include <cmath>
#include <random>
#include <stdexcept>
#include <unordered_map>

namespace fpb {

namespace {

struct Rng {  // mt19937_64 with explicit, library-independent mappings
  std::mt19937_64 g;
  explicit Rng(uint64_t s) : g(s) {}
  double uniform() { return double(g() >> 11) * 0x1.0p-53; }             // [0,1)
  double sym() { return 2.0 * uniform() - 1.0; }                          // [-1,1)
  double normal() {                                                       // Box-Muller
    const double u1 = 1.0 - uniform(), u2 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
  }
  double lognormal(double median, double s) { return s > 0 ? median * std::exp(s * normal()) : median; }
};

enum class Region : char { stick, slip, open };

using Face = FractureFace;
using Edge = FractureEdge;
using BcEdge = FractureBcEdge;

struct Mesh {
  int nn[3], nc[3];
  std::vector<std::array<double, 3>> nodes;
  std::vector<std::array<int, 8>> cells;
  std::vector<Face> faces;
  std::vector<Edge> edges;
  std::vector<BcEdge> bc_edges;
  std::vector<char> dir;  // per displacement dof
};

int tick_of(double x, double len, int cells, const char* what) {
  const double t = x / len * cells;
  const int i = int(std::lround(t));
  if (std::abs(t - i) > 1e-9 * std::max(1, cells)) throw std::invalid_argument(std::string(what) + ": not grid aligned");
  return i;
}

Mesh build_mesh(const WorkloadSpec& s) {
  Mesh m;
  for (int d = 0; d < 3; ++d) {
    if (s.cells[d] < 1) throw std::invalid_argument("build_mesh: axis with no cells");
    m.nc[d] = s.cells[d];
    m.nn[d] = s.cells[d] + 1;
  }
  auto tick = [&](int d, int i) { return s.length[d] * i / m.nc[d]; };  // AxisSpec::uniform (mesh.cpp:14-20)
  auto node_id = [&](int i, int j, int k) { return i + m.nn[0] * (j + m.nn[1] * k); };
  auto cell_id = [&](int i, int j, int k) { return i + m.nc[0] * (j + m.nc[1] * k); };
  m.nodes.reserve(size_t(m.nn[0]) * m.nn[1] * m.nn[2]);
  for (int k = 0; k < m.nn[2]; ++k)
    for (int j = 0; j < m.nn[1]; ++j)
      for (int i = 0; i < m.nn[0]; ++i) m.nodes.push_back({tick(0, i), tick(1, j), tick(2, k)});
  m.cells.resize(size_t(m.nc[0]) * m.nc[1] * m.nc[2]);
#pragma omp parallel for collapse(2)
  for (int k = 0; k < m.nc[2]; ++k)
    for (int j = 0; j < m.nc[1]; ++j)
      for (int i = 0; i < m.nc[0]; ++i)
        m.cells[cell_id(i, j, k)] = {node_id(i, j, k),         node_id(i + 1, j, k),     node_id(i + 1, j + 1, k),
                                     node_id(i, j + 1, k),     node_id(i, j, k + 1),     node_id(i + 1, j, k + 1),
                                     node_id(i + 1, j + 1, k + 1), node_id(i, j + 1, k + 1)};

  for (const FractureSpec& f : s.fractures) {  // mesh.cpp:77-179
    const int a = f.normal_axis, b = (a + 1) % 3, c = (a + 2) % 3;
    const int ia = tick_of(f.coord, s.length[a], m.nc[a], "fracture plane");
    if (ia == 0 || ia == m.nc[a]) throw std::invalid_argument("build_mesh: fracture plane on the boundary");
    const int jb0 = tick_of(f.lo1, s.length[b], m.nc[b], "fracture extent"),
              jb1 = tick_of(f.hi1, s.length[b], m.nc[b], "fracture extent"),
              jc0 = tick_of(f.lo2, s.length[c], m.nc[c], "fracture extent"),
              jc1 = tick_of(f.hi2, s.length[c], m.nc[c], "fracture extent");
    if (jb1 <= jb0 || jc1 <= jc0) throw std::invalid_argument("build_mesh: empty fracture patch");
    auto grid_node = [&](int jb, int jc) {
      int ijk[3];
      ijk[a] = ia, ijk[b] = jb, ijk[c] = jc;
      return node_id(ijk[0], ijk[1], ijk[2]);
    };
    std::unordered_map<int, int> dup;  // interior patch nodes are duplicated; the rim is shared
    for (int jb = jb0 + 1; jb < jb1; ++jb)
      for (int jc = jc0 + 1; jc < jc1; ++jc) {
        const int orig = grid_node(jb, jc);
        dup[orig] = int(m.nodes.size());
        m.nodes.push_back(m.nodes[orig]);
      }
    if (!dup.empty()) {  // the plus-side cell layer references the duplicates
      int lo[3] = {0, 0, 0}, hi[3] = {m.nc[0], m.nc[1], m.nc[2]};
      lo[a] = ia, hi[a] = ia + 1;
      for (int k = lo[2]; k < hi[2]; ++k)
        for (int j = lo[1]; j < hi[1]; ++j)
          for (int i = lo[0]; i < hi[0]; ++i)
            for (int& v : m.cells[cell_id(i, j, k)]) {
              auto it = dup.find(v);
              if (it != dup.end()) v = it->second;
            }
    }
    const int first = int(m.faces.size());
    for (int jc = jc0; jc < jc1; ++jc)
      for (int jb = jb0; jb < jb1; ++jb) {
        Face fc;
        fc.len1 = tick(b, jb + 1) - tick(b, jb);
        fc.len2 = tick(c, jc + 1) - tick(c, jc);
        fc.area = fc.len1 * fc.len2;
        fc.axis[0] = a, fc.axis[1] = b, fc.axis[2] = c;
        const int corner[4][2] = {{jb, jc}, {jb + 1, jc}, {jb + 1, jc + 1}, {jb, jc + 1}};
        for (int v = 0; v < 4; ++v) {
          const int orig = grid_node(corner[v][0], corner[v][1]);
          fc.minus[v] = orig;
          auto it = dup.find(orig);
          fc.plus[v] = it == dup.end() ? orig : it->second;
        }
        m.faces.push_back(fc);
      }
    const int nb = jb1 - jb0, ncc = jc1 - jc0;
    auto face_at = [&](int i1, int i2) { return first + i1 + nb * i2; };
    for (int i2 = 0; i2 < ncc; ++i2)
      for (int i1 = 0; i1 < nb; ++i1) {
        const Face& K = m.faces[face_at(i1, i2)];
        if (i1 + 1 < nb) {
          const Face& L = m.faces[face_at(i1 + 1, i2)];
          m.edges.push_back({face_at(i1, i2), face_at(i1 + 1, i2), K.len2, 0.5 * K.len1, 0.5 * L.len1});
        }
        if (i2 + 1 < ncc) {
          const Face& L = m.faces[face_at(i1, i2 + 1)];
          m.edges.push_back({face_at(i1, i2), face_at(i1, i2 + 1), K.len1, 0.5 * K.len2, 0.5 * L.len2});
        }
        const bool corner = (i1 == 0 || i1 == nb - 1) && (i2 == 0 || i2 == ncc - 1);
        if (!corner) continue;
        if (i1 == 0) m.bc_edges.push_back({face_at(i1, i2), K.len2, 0.5 * K.len1});
        if (i1 == nb - 1 && nb > 1) m.bc_edges.push_back({face_at(i1, i2), K.len2, 0.5 * K.len1});
        if (i2 == 0) m.bc_edges.push_back({face_at(i1, i2), K.len1, 0.5 * K.len2});
        if (i2 == ncc - 1 && ncc > 1) m.bc_edges.push_back({face_at(i1, i2), K.len1, 0.5 * K.len2});
      }
  }
  // Dirichlet base: zmin fixed (all three components); other faces free / loaded.
  m.dir.assign(3 * m.nodes.size(), 0);
  const double span = std::max(1.0, s.length[2]);
#pragma omp parallel for
  for (long v = 0; v < long(m.nodes.size()); ++v)
    if (std::abs(m.nodes[v][2] - 0.0) <= 1e-9 * span) m.dir[3 * v] = m.dir[3 * v + 1] = m.dir[3 * v + 2] = 1;
  return m;
}

const double kG = 1.0 / std::sqrt(3.0);
const double kXi[8] = {-1, 1, 1, -1, -1, 1, 1, -1};
const double kEta[8] = {-1, -1, 1, 1, -1, -1, 1, 1};
const double kZeta[8] = {-1, -1, -1, -1, 1, 1, 1, 1};

// 24x24 trilinear hexahedron stiffness, 2x2x2 Gauss (assembly.cpp:39-85)
void element_stiffness(const std::array<double, 3> xyz[8], double lambda, double mu, double ke[24][24]) {
  for (int i = 0; i < 24; ++i)
    for (int j = 0; j < 24; ++j) ke[i][j] = 0.0;
  for (int gp = 0; gp < 8; ++gp) {
    const double xi = kXi[gp] * kG, eta = kEta[gp] * kG, zeta = kZeta[gp] * kG;
    double dN[8][3];
    for (int a = 0; a < 8; ++a) {
      dN[a][0] = 0.125 * kXi[a] * (1 + kEta[a] * eta) * (1 + kZeta[a] * zeta);
      dN[a][1] = 0.125 * (1 + kXi[a] * xi) * kEta[a] * (1 + kZeta[a] * zeta);
      dN[a][2] = 0.125 * (1 + kXi[a] * xi) * (1 + kEta[a] * eta) * kZeta[a];
    }
    double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    for (int a = 0; a < 8; ++a)
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) J[r][c] += dN[a][r] * xyz[a][c];
    const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                       J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                       J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
    if (!(det > 0.0)) throw std::runtime_error("assemble_elasticity: degenerate cell Jacobian");
    double inv[3][3];
    inv[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) / det;
    inv[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
    inv[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
    inv[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) / det;
    inv[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
    inv[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
    inv[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) / det;
    inv[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
    inv[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
    double g[8][3];
    for (int a = 0; a < 8; ++a)
      for (int d = 0; d < 3; ++d) g[a][d] = inv[d][0] * dN[a][0] + inv[d][1] * dN[a][1] + inv[d][2] * dN[a][2];
    for (int a = 0; a < 8; ++a)
      for (int b = 0; b < 8; ++b) {
        const double gab = g[a][0] * g[b][0] + g[a][1] * g[b][1] + g[a][2] * g[b][2];
        for (int di = 0; di < 3; ++di)
          for (int dj = 0; dj < 3; ++dj) {
            double k = lambda * g[a][di] * g[b][dj];
            if (di == dj) k += mu * gab;
            k += mu * g[a][dj] * g[b][di];
            ke[3 * a + di][3 * b + dj] += k * det;
          }
      }
  }
}

}  // namespace

WorkloadSpec preset_config(int id, uint64_t seed) {
  WorkloadSpec s;
  s.seed = seed;
  auto cube = [&](int n) {
    s.cells[0] = s.cells[1] = s.cells[2] = n;
    s.length[0] = s.length[1] = s.length[2] = 1.0;
  };
  auto plane = [&](int axis, double c) {
    FractureSpec f;
    f.normal_axis = axis;
    f.coord = c;
    const int b = (axis + 1) % 3, cc = (axis + 2) % 3;
    f.lo1 = 0.0, f.hi1 = s.length[b], f.lo2 = 0.0, f.hi2 = s.length[cc];
    s.fractures.push_back(f);
  };
  switch (id) {
    case 1:  // 20^3, one vertical fracture at x = 0.5; homogeneous E; 70/20/10
      cube(20);
      plane(0, 0.5);
      s.frac_stick = 0.7, s.frac_slip = 0.2;
      break;
    case 2:  // 40^3, one fracture; lognormal E (0.5) and aperture (0.3); 60/30/10
      cube(40);
      plane(0, 0.5);
      s.E_sigma_ln = 0.5, s.aperture_sigma_ln = 0.3;
      s.frac_stick = 0.6, s.frac_slip = 0.3;
      break;
    case 3:  // 80^3, three parallel vertical fractures
      cube(80);
      plane(0, 0.25), plane(0, 0.5), plane(0, 0.75);
      s.E_sigma_ln = 0.5, s.aperture_sigma_ln = 0.3;
      s.frac_stick = 0.6, s.frac_slip = 0.3;
      break;
    case 4:  // 100^3, 10 full orthogonal planes (4 x, 3 y, 3 z); E sigma_ln 1.0; 50/40/10
      cube(100);
      for (double c : {0.2, 0.4, 0.6, 0.8}) plane(0, c);
      for (double c : {0.25, 0.5, 0.75}) plane(1, c);
      for (double c : {0.25, 0.5, 0.75}) plane(2, c);
      s.E_sigma_ln = 1.0, s.aperture_sigma_ln = 0.3;
      s.frac_stick = 0.5, s.frac_slip = 0.4;
      break;
    case 5: {  // 256x256x128, 16 stiffness layers, 40 random axis-aligned rectangles (32..128 faces)
      s.cells[0] = 256, s.cells[1] = 256, s.cells[2] = 128;
      s.length[0] = 2.0, s.length[1] = 2.0, s.length[2] = 1.0;
      s.E_sigma_ln = 1.0, s.E_layers = 16, s.nu_lo = 0.2, s.nu_hi = 0.3;
      s.aperture_sigma_ln = 0.5;
      s.frac_stick = 0.6, s.frac_slip = 0.3;
      Rng r(seed ^ 0x5eedf00dULL);
      std::vector<std::vector<int>> used(3);
      while (s.fractures.size() < 40) {
        const int axis = int(r.g() % 3), b = (axis + 1) % 3, c = (axis + 2) % 3;
        const int ia = 1 + int(r.g() % uint64_t(s.cells[axis] - 1));
        if (std::find(used[axis].begin(), used[axis].end(), ia) != used[axis].end()) continue;
        const int w1 = std::min(s.cells[b], 32 + int(r.g() % 97)), w2 = std::min(s.cells[c], 32 + int(r.g() % 97));
        const int o1 = int(r.g() % uint64_t(s.cells[b] - w1 + 1)), o2 = int(r.g() % uint64_t(s.cells[c] - w2 + 1));
        used[axis].push_back(ia);
        FractureSpec f;
        f.normal_axis = axis;
        f.coord = s.length[axis] * ia / s.cells[axis];
        f.lo1 = s.length[b] * o1 / s.cells[b], f.hi1 = s.length[b] * (o1 + w1) / s.cells[b];
        f.lo2 = s.length[c] * o2 / s.cells[c], f.hi2 = s.length[c] * (o2 + w2) / s.cells[c];
        s.fractures.push_back(f);
      }
      break;
    }
    default:
      throw std::invalid_argument("preset_config: config id must be 1..5");
  }
  return s;
}

// assemble_fracture_blocks (assembly.cpp:229-406): C2 (jump rows, slip derivative), H (stabilization and
// the slip / open diagonal), T (TPFA, cubic law, stabilization / dt), F_u (pressure-gap coupling) and
// Q2 = Q2gap + F_u, every block through from_triplets in insertion order
void assemble_fracture_blocks(const FractureModel& M, const FractureState& S, HostSystem& J) {
  const int n_u = M.n_u, n_p = M.n_p, n_t = 3 * n_p;
  if (int(S.region.size()) != n_p || int(S.gap.size()) != n_p || int(S.trac_n.size()) != n_p ||
      int(S.slip_dir.size()) != n_p || int(S.pressure.size()) != n_p)
    throw std::invalid_argument("assemble_fracture_blocks: state size != n_p");
  std::vector<Csr::Triplet> c2, h, t, q2gap, fu;
  auto jump_row = [&](int f, int row, int comp, double scale) {
    const Face& fc = M.faces[f];
    const double w = fc.area / 4.0;
    for (int v = 0; v < 4; ++v) {
      if (fc.plus[v] == fc.minus[v]) continue;
      for (int d = 0; d < 3; ++d) {
        const double val = scale * w * (fc.axis[comp] == d ? 1.0 : 0.0);
        if (val == 0.0) continue;
        const int cp = 3 * fc.plus[v] + d, cm = 3 * fc.minus[v] + d;
        if (!M.dir[cp]) c2.push_back({row, cp, val});
        if (!M.dir[cm]) c2.push_back({row, cm, -val});
      }
    }
  };
  for (int f = 0; f < n_p; ++f) {
    const Face& fc = M.faces[f];
    if (S.region[f] == 's') {
      for (int c = 0; c < 3; ++c) jump_row(f, 3 * f + c, c, 1.0);
    } else if (S.region[f] == 'l') {
      jump_row(f, 3 * f, 0, 1.0);
      const double dg[2] = {S.gap[f][1], S.gap[f][2]};  // gap_prev = 0
      // |dg_T| (std::hypot at assembly.cpp:271): the square root of the sum, so the device assembly
      // reproduces it bit for bit (CUDA's and glibc's hypot differ in the last bit; a 1-ulp change)
      const double r = std::sqrt(dg[0] * dg[0] + dg[1] * dg[1]);
      const double tau = M.cohesion - S.trac_n[f] * M.tan_th;
      const double thr = std::max(1e-12, 0.1 * std::max(tau, 0.0) / M.k_scale);
      double mm[2], D[2][2] = {{0, 0}, {0, 0}};
      if (r >= thr) {
        mm[0] = dg[0] / r, mm[1] = dg[1] / r;
        for (int a = 0; a < 2; ++a)
          for (int b = 0; b < 2; ++b) D[a][b] = (tau / r) * ((a == b ? 1.0 : 0.0) - mm[a] * mm[b]);
      } else {
        mm[0] = S.slip_dir[f][0], mm[1] = S.slip_dir[f][1];
      }
      for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b)
          if (D[a][b] != 0.0) jump_row(f, 3 * f + 1 + a, 1 + b, -D[a][b] / M.k_scale);
      for (int a = 0; a < 2; ++a) {
        h.push_back({3 * f + 1 + a, 3 * f + 1 + a, -fc.area / M.k_scale});
        const double dtn = -M.tan_th * mm[a];
        if (dtn != 0.0) h.push_back({3 * f + 1 + a, 3 * f, (fc.area / M.k_scale) * dtn});
      }
    } else {
      for (int c = 0; c < 3; ++c) h.push_back({3 * f + c, 3 * f + c, -fc.area / M.k_scale});
    }
  }
  auto stab = [&](const Edge& e) {  // beta * (mean face area / E) * |edge| (assembly.cpp:94-97)
    const double hh = 0.5 * (M.faces[e.k].area + M.faces[e.l].area);
    return M.stab_beta * (hh / M.E_ref) * e.length;
  };
  for (const Edge& e : M.edges) {
    const bool ck = S.region[e.k] != 'o', cl = S.region[e.l] != 'o';
    if (!ck && !cl) continue;
    const double sc = stab(e);
    for (int c = 0; c < 3; ++c) {
      if (ck && cl) {
        h.push_back({3 * e.k + c, 3 * e.k + c, sc});
        h.push_back({3 * e.l + c, 3 * e.l + c, sc});
        h.push_back({3 * e.k + c, 3 * e.l + c, -sc});
        h.push_back({3 * e.l + c, 3 * e.k + c, -sc});
      } else if (ck) {
        h.push_back({3 * e.k + c, 3 * e.k + c, sc});
      } else {
        h.push_back({3 * e.l + c, 3 * e.l + c, sc});
      }
    }
  }
  std::vector<double> cf(static_cast<size_t>(n_p)), dcf(static_cast<size_t>(n_p));
  for (int f = 0; f < n_p; ++f) {
    const bool open = S.region[f] == 'o';
    const double g = open ? std::max(S.gap[f][0], 0.0) : 0.0;
    cf[f] = M.C_f0 + g * g * g / 12.0;
    dcf[f] = open ? g * g / 4.0 : 0.0;
  }
  auto fu_row = [&](int row, int face, double coeff) {
    if (coeff == 0.0) return;
    const Face& fc = M.faces[face];
    for (int v = 0; v < 4; ++v) {
      if (fc.plus[v] == fc.minus[v]) continue;
      for (int d = 0; d < 3; ++d) {
        const double val = coeff * (fc.axis[0] == d ? 1.0 : 0.0) / 4.0;
        if (val == 0.0) continue;
        const int cp = 3 * fc.plus[v] + d, cm = 3 * fc.minus[v] + d;
        if (!M.dir[cp]) fu.push_back({row, cp, val});
        if (!M.dir[cm]) fu.push_back({row, cm, -val});
      }
    }
  };
  for (const Edge& e : M.edges) {
    const double yk = (cf[e.k] / M.mu_f) * e.length / e.dk, yl = (cf[e.l] / M.mu_f) * e.length / e.dl;
    const double ykl = 2.0 * yk * yl / (yk + yl);
    t.push_back({e.k, e.k, ykl});
    t.push_back({e.l, e.l, ykl});
    t.push_back({e.k, e.l, -ykl});
    t.push_back({e.l, e.k, -ykl});
    const double sc = stab(e) / M.dt;
    t.push_back({e.k, e.k, sc});
    t.push_back({e.l, e.l, sc});
    t.push_back({e.k, e.l, -sc});
    t.push_back({e.l, e.k, -sc});
    const double dp = S.pressure[e.k] - S.pressure[e.l];
    if (dp != 0.0) {
      const double dk = 2.0 * (yl / (yk + yl)) * (yl / (yk + yl)), dl = 2.0 * (yk / (yk + yl)) * (yk / (yk + yl));
      const double ck = dp * dk * (e.length / (M.mu_f * e.dk)) * dcf[e.k];
      const double cl = dp * dl * (e.length / (M.mu_f * e.dl)) * dcf[e.l];
      fu_row(e.k, e.k, ck);
      fu_row(e.k, e.l, cl);
      fu_row(e.l, e.k, -ck);
      fu_row(e.l, e.l, -cl);
    }
  }
  for (const BcEdge& e : M.bc_edges) {
    const double yb = (cf[e.k] / M.mu_f) * e.length / e.d;
    t.push_back({e.k, e.k, yb});
    const double pk = S.pressure[e.k];
    if (pk != 0.0) fu_row(e.k, e.k, pk * (e.length / (M.mu_f * e.d)) * dcf[e.k]);
  }
  for (int f = 0; f < n_p; ++f) {
    if (S.region[f] != 'o') continue;
    const Face& fc = M.faces[f];
    const double w = fc.area / 4.0;
    for (int v = 0; v < 4; ++v) {
      if (fc.plus[v] == fc.minus[v]) continue;
      for (int d = 0; d < 3; ++d) {
        const double val = (w / M.dt) * (fc.axis[0] == d ? 1.0 : 0.0);
        if (val == 0.0) continue;
        const int cp = 3 * fc.plus[v] + d, cm = 3 * fc.minus[v] + d;
        if (!M.dir[cp]) q2gap.push_back({f, cp, val});
        if (!M.dir[cm]) q2gap.push_back({f, cm, -val});
      }
    }
  }
  J.C2 = Csr::from_triplets(n_t, n_u, std::move(c2));
  J.H = Csr::from_triplets(n_t, n_t, std::move(h));
  J.T = Csr::from_triplets(n_p, n_p, std::move(t));
  J.F_u = Csr::from_triplets(n_p, n_u, std::move(fu));
  J.Q2 = csr_add(Csr::from_triplets(n_p, n_u, std::move(q2gap)), J.F_u, 1.0, 1.0);
}

Workload generate_workload(const WorkloadSpec& s) {
  Mesh m = build_mesh(s);
  const int n_nodes = int(m.nodes.size()), n_u = 3 * n_nodes, n_p = int(m.faces.size()), n_t = 3 * n_p;
  Workload W;
  W.n_fractures = int(s.fractures.size());
  W.coords = m.nodes;
  HostSystem& J = W.J;
  J.n_u = n_u, J.n_t = n_t, J.n_p = n_p;

  // ---- per-cell materials
  const size_t n_cells = m.cells.size();
  std::vector<double> lam(n_cells), mu(n_cells);
  {
    Rng r(s.seed * 0x9e3779b97f4a7c15ULL + 1);
    std::vector<double> layer_E, layer_nu;
    if (s.E_layers > 0)
      for (int l = 0; l < s.E_layers; ++l) {
        layer_E.push_back(r.lognormal(s.E_median, s.E_sigma_ln));
        layer_nu.push_back(s.nu_hi > s.nu_lo ? s.nu_lo + (s.nu_hi - s.nu_lo) * r.uniform() : s.nu);
      }
    for (size_t c = 0; c < n_cells; ++c) {
      double E, nu = s.nu;
      if (s.E_layers > 0) {
        const int kz = int(c / (size_t(m.nc[0]) * m.nc[1]));
        const int l = std::min(s.E_layers - 1, kz * s.E_layers / m.nc[2]);
        E = layer_E[l], nu = layer_nu[l];
      } else {
        E = r.lognormal(s.E_median, s.E_sigma_ln);
      }
      lam[c] = E * nu / ((1 + nu) * (1 - 2 * nu));
      mu[c] = E / (2 * (1 + nu));
    }
  }
  const double E_ref = s.E_median;  // stab_scalar and k_scale use one modulus (the median)

  // ---- node graph and the 3x3-block pattern of A (assembly.cpp:138-159)
  std::vector<int64_t> nc_off(static_cast<size_t>(n_nodes) + 1, 0);
  for (const auto& cell : m.cells)
    for (int v : cell) ++nc_off[size_t(v) + 1];
  for (int v = 0; v < n_nodes; ++v) nc_off[size_t(v) + 1] += nc_off[v];
  std::vector<int> node_cells(static_cast<size_t>(nc_off[n_nodes]));
  {
    std::vector<int64_t> next(nc_off.begin(), nc_off.end() - 1);
    for (size_t c = 0; c < n_cells; ++c)
      for (int v : m.cells[c]) node_cells[next[v]++] = int(c);
  }
  std::vector<std::vector<int>> nbr(static_cast<size_t>(n_nodes));
#pragma omp parallel for schedule(dynamic, 1024)
  for (int v = 0; v < n_nodes; ++v) {
    auto& L = nbr[v];
    for (int64_t q = nc_off[v]; q < nc_off[v + 1]; ++q)
      for (int w : m.cells[node_cells[q]]) L.push_back(w);
    std::sort(L.begin(), L.end());
    L.erase(std::unique(L.begin(), L.end()), L.end());
  }
  Csr& A = J.A;
  A = Csr(n_u, n_u);
  for (int v = 0; v < n_nodes; ++v)
    for (int d = 0; d < 3; ++d) A.rp[3 * size_t(v) + d + 1] = A.rp[3 * size_t(v) + d] + 3 * int64_t(nbr[v].size());
  A.ci.resize(static_cast<size_t>(A.rp[n_u]));
  A.v.assign(static_cast<size_t>(A.rp[n_u]), 0.0);
#pragma omp parallel for schedule(dynamic, 1024)
  for (int v = 0; v < n_nodes; ++v)
    for (int d = 0; d < 3; ++d) {
      int64_t p = A.rp[3 * size_t(v) + d];
      for (int w : nbr[v])
        for (int e = 0; e < 3; ++e) A.ci[p++] = 3 * w + e;
    }
  // ---- stiffness scatter, 8 parity colors so concurrent cells never share a node
  for (int color = 0; color < 8; ++color) {
#pragma omp parallel for schedule(dynamic, 256)
    for (long c = 0; c < long(n_cells); ++c) {
      const int ci = int(c % m.nc[0]), cj = int((c / m.nc[0]) % m.nc[1]), ck = int(c / (size_t(m.nc[0]) * m.nc[1]));
      if (((ci & 1) | ((cj & 1) << 1) | ((ck & 1) << 2)) != color) continue;
      const auto& cell = m.cells[c];
      std::array<double, 3> xyz[8];
      for (int a = 0; a < 8; ++a) xyz[a] = m.nodes[cell[a]];
      double ke[24][24];
      element_stiffness(xyz, lam[c], mu[c], ke);
      for (int a = 0; a < 8; ++a) {
        const auto& L = nbr[cell[a]];
        for (int b = 0; b < 8; ++b) {
          const int slot = int(std::lower_bound(L.begin(), L.end(), cell[b]) - L.begin());
          for (int di = 0; di < 3; ++di) {
            const int64_t base = A.rp[3 * size_t(cell[a]) + di] + 3 * slot;
            for (int dj = 0; dj < 3; ++dj) A.v[base + dj] += ke[3 * a + di][3 * b + dj];
          }
        }
      }
    }
  }
  // symmetric Dirichlet elimination with unit diagonal (assembly.cpp:179-186)
#pragma omp parallel for schedule(static)
  for (int row = 0; row < n_u; ++row) {
    const bool rd = m.dir[row];
    for (int64_t k = A.rp[row]; k < A.rp[row + 1]; ++k) {
      const int col = A.ci[k];
      if (rd || m.dir[col]) A.v[k] = row == col ? 1.0 : 0.0;
    }
  }

  // ---- fracture state (seeded)
  double mean_h = 0.0;
  for (const Face& f : m.faces) mean_h += std::sqrt(f.area);
  mean_h = n_p > 0 ? mean_h / n_p : 0.0;
  const double k_scale = mean_h > 0 ? E_ref / mean_h : E_ref;  // assembly.cpp:87-91
  W.k_scale = k_scale;
  const double tan_th = s.friction;  // theta = atan(mu)
  std::vector<Region> region(static_cast<size_t>(n_p));
  std::vector<std::array<double, 3>> gap(static_cast<size_t>(n_p), {0, 0, 0}), trac(static_cast<size_t>(n_p), {0, 0, 0});
  std::vector<double> pres(static_cast<size_t>(n_p), 0.0);
  std::vector<std::array<double, 2>> sdir(static_cast<size_t>(n_p), {1.0, 0.0});
  {
    Rng r(s.seed * 0xbf58476d1ce4e5b9ULL + 7);
    for (int f = 0; f < n_p; ++f) {
      const double u = r.uniform();
      region[f] = u < s.frac_stick ? Region::stick : (u < s.frac_stick + s.frac_slip ? Region::slip : Region::open);
      trac[f][0] = -s.sigma_load * (1.0 + 0.1 * r.sym());
      pres[f] = s.p0 * (1.0 + 0.1 * r.sym());
      const double ap = r.lognormal(s.aperture_median, s.aperture_sigma_ln);
      const double phi = 6.283185307179586 * r.uniform(), mag = 1.0 + r.uniform();
      if (region[f] == Region::open) gap[f][0] = ap;
      if (region[f] == Region::slip) {
        const double tau = s.cohesion - trac[f][0] * tan_th;
        const double thr = std::max(1e-12, 0.1 * std::max(tau, 0.0) / k_scale);
        gap[f][1] = s.slip_factor * thr * mag * std::cos(phi);
        gap[f][2] = s.slip_factor * thr * mag * std::sin(phi);
        sdir[f] = {std::cos(phi), std::sin(phi)};
      }
    }
    for (Region q : region) (q == Region::stick ? W.n_stick : q == Region::slip ? W.n_slip : W.n_open)++;
    W.region.reserve(region.size());
    for (Region q : region) W.region.push_back(q == Region::stick ? 's' : q == Region::slip ? 'l' : 'o');
    W.dt = s.dt;
  }

  // ---- coupling C1, Q1 (assembly.cpp:190-216)
  std::vector<Csr::Triplet> c1, q1;
  for (int f = 0; f < n_p; ++f) {
    const Face& fc = m.faces[f];
    const double w = fc.area / 4.0;
    for (int v = 0; v < 4; ++v) {
      if (fc.plus[v] == fc.minus[v]) continue;
      for (int side = 0; side < 2; ++side) {
        const int node = side == 0 ? fc.plus[v] : fc.minus[v];
        const double sgn = side == 0 ? 1.0 : -1.0;
        for (int d = 0; d < 3; ++d) {
          const int row = 3 * node + d;
          if (m.dir[row]) continue;
          for (int c = 0; c < 3; ++c) {
            const double val = sgn * w * (fc.axis[c] == d ? 1.0 : 0.0);
            if (val != 0.0) c1.push_back({row, 3 * f + c, val});
          }
          const double qv = -sgn * w * (fc.axis[0] == d ? 1.0 : 0.0);
          if (qv != 0.0) q1.push_back({row, f, qv});
        }
      }
    }
  }
  J.C1 = Csr::from_triplets(n_u, n_t, std::move(c1));
  J.Q1 = Csr::from_triplets(n_u, n_p, std::move(q1));

  // ---- state-dependent blocks (assembly.cpp:229-406)
  FractureModel& M = W.model;
  M.n_u = n_u, M.n_p = n_p;
  M.faces = m.faces, M.edges = m.edges, M.bc_edges = m.bc_edges, M.dir = m.dir;
  M.cohesion = s.cohesion, M.tan_th = tan_th, M.k_scale = k_scale, M.stab_beta = s.stab_beta, M.E_ref = E_ref;
  M.C_f0 = s.C_f0, M.mu_f = s.mu_f, M.dt = s.dt;
  FractureState& S = W.state;
  S.region = W.region;
  S.gap = gap;
  S.trac_n.resize(static_cast<size_t>(n_p));
  for (int f = 0; f < n_p; ++f) S.trac_n[f] = trac[f][0];
  S.slip_dir = sdir;
  S.pressure = pres;
  assemble_fracture_blocks(M, S, J);
  J.check_shapes();
  return W;
}

}  // namespace fpb
