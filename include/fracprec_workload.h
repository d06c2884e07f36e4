/*
 * fracprec workload generator (libfp_workload.so, workload/) — synthetic inputs
 * for the BASELINE.json configs (structured hex mesh with duplicated fracture
 * nodes, trilinear elasticity, TPFA fracture flow, seeded contact state) and
 * the snapshot bundle reader/writer.  Restates the reference's input side
 * (/root/reference/proj/core/src/mesh.cpp, assembly.cpp, snapshot.cpp, mmio.cpp),
 * which is not on the solve path.  A host-only library of its own: the B200
 * solve library and the CPU oracle's callers both build the same systems from
 * it, and the oracle-side callers never load the solve library.
 *
 * Only the data types of fracprec_b200.h are used (no link dependency).  Status
 * codes are FP_*; fp_workload_last_error() gives this library's message.
 */
#ifndef FRACPREC_WORKLOAD_H
#define FRACPREC_WORKLOAD_H

#include <stdint.h>

#include "fracprec_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fp_fracture_spec { /* FractureSpec (mesh.hpp:28-33) */
  int32_t normal_axis;
  double coord, lo1, hi1, lo2, hi2;
} fp_fracture_spec;

typedef struct fp_workload_spec {
  int32_t cells[3];
  double length[3];
  int32_t n_fractures;
  const fp_fracture_spec* fractures;
  double E_median, E_sigma_ln;
  int32_t E_layers;
  double nu, nu_lo, nu_hi;
  double frac_stick, frac_slip;
  double aperture_median, aperture_sigma_ln;
  uint64_t seed;
  double stab_beta;  /* jump-penalty constant (assembly.hpp:26 / presets.cpp:246); <= 0 selects the preset value */
  double slip_factor; /* slip increment in units of the 0.1 tau/k freeze threshold; <= 0 selects the preset value */
} fp_workload_spec;

typedef struct fp_workload fp_workload;

const char* fp_workload_last_error(void);
/* layout fingerprint of the C++ handle types (workload/workload.hpp): the solve library checks it */
uint64_t fp_workload_layout(void);

/* config_id 1..5 = BASELINE.json configs[0..4] */
int fp_workload_preset(int32_t config_id, uint64_t seed, fp_workload** out);
int fp_workload_custom(const fp_workload_spec* spec, fp_workload** out);
void fp_workload_destroy(fp_workload* w);
/* views into the workload's arrays (64-bit row offsets), valid until destroy */
int fp_workload_system(const fp_workload* w, fp_block_system* J);
int fp_workload_coords(const fp_workload* w, const double** xyz, int32_t* n_nodes);
/* counts[0..3] = stick, slip, open, fractures */
int fp_workload_info(const fp_workload* w, int32_t* counts);
/* per-face contact state ('s' stick, 'l' slip, 'o' open; Snapshot::region_string, snapshot.cpp:20-25)
 * and the time step; the string is valid until destroy */
int fp_workload_region(const fp_workload* w, const char** region, double* dt);

/* FractureState (assembly.hpp) of a workload: per face the contact region, the gap increment (normal,
 * m1, m2), the normal traction, the frozen slip direction and the pressure */
typedef struct fp_fracture_state {
  int32_t n_p;
  const char* region;        /* n_p characters: 's' stick, 'l' slip, 'o' open */
  const double* gap;         /* 3 n_p */
  const double* traction_n;  /* n_p */
  const double* slip_dir;    /* 2 n_p */
  const double* pressure;    /* n_p */
} fp_fracture_state;
/* views of the workload's current state (valid until the next set_state or destroy) */
int fp_workload_state(const fp_workload* w, fp_fracture_state* out);
/* a new state: C2, H, T, F_u, Q2 re-assembled on the host (assemble_fracture_blocks, assembly.cpp:229-406),
 * the reference's Newton-step assembly; fp_workload_system views see the new blocks */
int fp_workload_set_state(fp_workload* w, const fp_fracture_state* st);

/* ---- snapshot bundle (snapshot.cpp:28-104, mmio.cpp:15-76): manifest.json + Matrix Market blocks */
/* import_snapshot: the bundle in `dir` as a workload handle (system views, coords, region, dt) */
int fp_snapshot_import(const char* dir, fp_workload** out);
/* export_snapshot: region = n_p characters s/l/o; node_coords may be null (n_nodes = 0) */
int fp_snapshot_export(const char* dir, const fp_block_system* J, const char* region, double dt,
                       const double* node_coords, int32_t n_nodes);

#ifdef __cplusplus
}
#endif

#endif
