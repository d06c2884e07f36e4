// Snapshot bundle I/O: the reference's on-disk interchange for a Jacobian
// (/root/reference/proj/core/src/snapshot.cpp:28-104, mmio.cpp:15-76): the
// seven blocks plus F_u as Matrix Market files, sizes / region labels / dt in
// manifest.json, optional node coordinates as a text vector.  This feeds real
// driver states to the GPU solve.
//
// B200-host design: files are read whole and parsed in parallel (token counts
// per chunk, then a prefix sum assigns every token its (entry, field) slot),
// numbers go through std::from_chars (correctly rounded, like the stream
// extraction the reference uses); CSR assembly keeps from_triplets' semantics
// (stable (row, col) order, duplicates summed from 0.0 in file order).  The
// writer formats rows in parallel with the reference's exact printf formats.
#pragma once

#include <array>
#include <string>
#include <vector>

#include "workload.hpp"

namespace fpb {

Csr read_matrix_market(const std::string& path);                    // mmio.cpp:15-48
void write_matrix_market(const std::string& path, const Csr& A);    // mmio.cpp:50-59
std::vector<double> read_vector_text(const std::string& path);      // mmio.cpp:61-69
void write_vector_text(const std::string& path, const std::vector<double>& v);  // mmio.cpp:71-76

// import_snapshot (snapshot.cpp:67-104) into a Workload (system, coords, region labels, dt)
Workload import_snapshot(const std::string& dir);
// export_snapshot (snapshot.cpp:28-65); region: n_p characters 's' / 'l' / 'o'
void export_snapshot(const std::string& dir, const HostSystem& J, const std::string& region, double dt,
                     const std::vector<std::array<double, 3>>& coords);

}  // namespace fpb
