// Synthetic workload generator for the BASELINE.json configs: a restatement of
// the reference's structured-hex mesh with duplicated fracture nodes
// (/root/reference/proj/core/src/mesh.cpp:51-224) and its Jacobian assembly
// (assembly.cpp:39-97,132-406), extended with per-cell Young's modulus and
// Poisson ratio (BASELINE configs 2-5) and a seeded FractureState.  This is input
// generation for the solve path, not part of it.
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "wcsr.hpp"

namespace fpb {

struct FractureSpec {  // mesh.hpp:28-33
  int normal_axis = 0;
  double coord = 0, lo1 = 0, hi1 = 0, lo2 = 0, hi2 = 0;
};

struct WorkloadSpec {
  int cells[3] = {20, 20, 20};
  double length[3] = {1.0, 1.0, 1.0};
  std::vector<FractureSpec> fractures;
  // elasticity (per cell): E lognormal(median, sigma_ln) per element or per z-layer
  double E_median = 10e9, E_sigma_ln = 0.0;
  int E_layers = 0;                 // 0: independent per element; >0: per z-layer
  double nu = 0.25, nu_lo = 0.0, nu_hi = 0.0;  // nu_hi > nu_lo: per-layer U(nu_lo, nu_hi)
  // contact / flow (assembly.hpp:18-39)
  // stab_beta = 1.0: the reference's value for problems read from JSON (presets.cpp:246).  Its struct
  // default 0.02 (assembly.hpp:26) makes the stick penalty C1 H~^-1 C2 50x stiffer and the
  // AMG-preconditioned solve stagnates ("Workload").
  double friction = 0.6, cohesion = 0.0, C_f0 = 9.87e-15, mu_f = 1e-3, stab_beta = 1.0, dt = 0.5;
  double frac_stick = 0.7, frac_slip = 0.2;  // open = rest
  double aperture_median = 1e-4, aperture_sigma_ln = 0.0;
  // slip increment |dg_T| = slip_factor * (0.1 tau / k) * (1 + U[0,1)): SURVEY §8(d) asks for >= 10x the
  // direction-freeze threshold of assembly.cpp:20-23 so that dt_T/dg_T = (tau/|dg_T|)(I - m m^T) != 0
  double slip_factor = 10.0;
  double sigma_load = 1e7;  // top-face compressive load, Pa
  double p0 = 1e6;          // fracture pressure level, Pa
  uint64_t seed = 42;
};

// The fixed part of the state-dependent assembly (assemble_fracture_blocks, assembly.cpp:229-406): the
// fracture faces (minus / plus nodes, area, frame), the TPFA edges between faces and to the patch rim,
// the Dirichlet flags of the displacement dofs and the material constants.
struct FractureFace {
  int minus[4], plus[4];
  double area, len1, len2;
  int axis[3];  // frame: normal axis, m1 axis, m2 axis (unit vectors e_axis)
};
struct FractureEdge {
  int k, l;
  double length, dk, dl;
};
struct FractureBcEdge {
  int k;
  double length, d;
};
struct FractureModel {
  int n_u = 0, n_p = 0;
  std::vector<FractureFace> faces;
  std::vector<FractureEdge> edges;
  std::vector<FractureBcEdge> bc_edges;
  std::vector<char> dir;  // per displacement dof
  double cohesion = 0.0, tan_th = 0.6, k_scale = 1.0, stab_beta = 1.0, E_ref = 1.0, C_f0 = 9.87e-15, mu_f = 1e-3,
         dt = 0.5;
};
// FractureState (assembly.hpp): per face the contact region ('s' stick, 'l' slip, 'o' open), the gap
// increment (normal, m1, m2; the previous gap is 0), the normal traction, the frozen slip direction and
// the pressure
struct FractureState {
  std::string region;
  std::vector<std::array<double, 3>> gap;
  std::vector<double> trac_n;
  std::vector<std::array<double, 2>> slip_dir;
  std::vector<double> pressure;
};
// C2, H, T, F_u and Q2 of J for a state (the reference's Newton-step assembly; the generator's own)
void assemble_fracture_blocks(const FractureModel& M, const FractureState& S, HostSystem& J);

struct Workload {
  HostSystem J;
  FractureModel model;
  FractureState state;
  std::vector<std::array<double, 3>> coords;
  int n_stick = 0, n_slip = 0, n_open = 0, n_fractures = 0;
  double k_scale = 0.0;
  std::string region;  // per face 's' stick, 'l' slip, 'o' open (Snapshot::region_string, snapshot.cpp:20-25)
  double dt = 0.5;
};

WorkloadSpec preset_config(int config_id, uint64_t seed);  // BASELINE.json configs[0..4] as 1..5
Workload generate_workload(const WorkloadSpec& spec);

}  // namespace fpb

// the C ABI's opaque workload handle (include/fracprec_workload.h), shared with the solve library
struct fp_workload {
  fpb::Workload w;
};

// Layout fingerprint of the shared handle types: the solve library reads fp_workload's members directly
// (it is built against this header), so it checks at use that the loaded generator library was built
// from the same header (fp_workload_layout, include/fracprec_workload.h)
constexpr unsigned long long workload_layout_fingerprint() {
  return (unsigned long long)sizeof(fpb::Workload) ^ ((unsigned long long)sizeof(fpb::FractureModel) << 16) ^
         ((unsigned long long)sizeof(fpb::FractureState) << 32) ^ ((unsigned long long)sizeof(fpb::HostSystem) << 48);
}
