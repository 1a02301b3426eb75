// General (adaptive) meshes on the device — SURVEY §8f rows 2 and 3.
//
// The forest itself (refine with the 2:1 face-balance closure, cell ids in creation order,
// mesh.cpp:18-223) is host bookkeeping; everything per vertex / cell / dof runs on the device:
// the DofMap (sorted packed corner keys, fem.cpp:98-116), point location in the forest, the
// hanging-node + Dirichlet + active-set constraints with their closure (fem.cpp:148-267), the
// element loops with each cell's own edge h, the condensation through constraint masters and
// Eigen's setFromTriplets as precomputed "plans" (model.cpp:66-322), the Newton step, TCV/COD,
// the jump estimator, marking and transfer (adapt.cpp, fem.cpp:318-333).
#pragma once

#include <vector>

#include "cf_types.hpp"
#include "cf_vec.hpp"

namespace cfb {

constexpr int kLevelBits = 16;
constexpr i64 kUnit = i64(1) << kLevelBits;

struct HostCell {
  int level = 0;
  i64 anchor[3] = {0, 0, 0};
  int parent = -1;
  int child[8] = {-1, -1, -1, -1, -1, -1, -1, -1};
  bool active = true;
  i64 isize() const { return kUnit >> level; }
};

// device mirror of the forest (point location)
struct DevForest {
  int d = 2, n0 = 1, nroots = 0;
  const int* level = nullptr;
  const i64* anchor = nullptr;  // 3 per cell
  const int* child = nullptr;   // 8 per cell
  const std::uint8_t* active = nullptr;
  const int* roots = nullptr;
};

// scatter plan of one output (vector or CSR block): for output slot t, the ordered sources
// src[ptr[t] .. ptr[t+1]) with weights w (the condensation weight product, 1 for direct entries)
struct Plan {
  i64 n = 0;         // output slots (dofs, or (row, col) entries)
  DevBuf<i64> ptr;   // n + 1
  DevBuf<i64> src;   // indices into the per-cell element array
  DevBuf<double> w;
  DevBuf<int> row, col;  // CSR plans: the (row, column) of every slot (rows ascending, columns ascending)
  DevBuf<i64> rptr;      // CSR plans: first slot of every row (rows + 1)
  i64 rows = 0, cols = 0;
};

struct MeshDisc {
  // forest (host)
  int d = 2, n0 = 1;
  double K = 1.0, unit = 0.0;
  std::vector<HostCell> cells;
  std::vector<int> roots;
  std::vector<int> active;  // active ids, ascending (mesh.cpp:36-44)
  std::uint64_t revision = 0;
  // device forest + DofMap
  DevBuf<int> t_level, t_child, t_roots;
  DevBuf<i64> t_anchor;
  DevBuf<std::uint8_t> t_active;
  i64 V = 0, nact = 0;
  int max_level = 0;
  DevBuf<i64> vkey;   // sorted packed vertex keys (fem.cpp:100-116)
  DevBuf<int> cvert;  // active cell position -> 2^d vertex ids (z-order corners)
  DevBuf<int> clevel; // active cell position -> level
  DevBuf<int> cid;    // active cell position -> cell id
  // element tables per level (gp = G / h etc. for the cell's own h)
  std::vector<Tables> host_tabs;
  DevBuf<Tables> tabs;
  double tab_mu = -1.0, tab_lam = -1.0;
  // base-constraint plans (built with the first base constraint set of this mesh)
  bool plans_ready = false;
  std::uint64_t plan_uid = 0;  // the constraint set the plans were built from
  Plan res;          // residual: slot = dof
  Plan uu, pu, pp;   // Jacobian entries
  Plan self;         // dof -> its own (cell, local dof) incidences (constrained diagonals)
  // the base constraint set of the Newton step (Dirichlet clamp + hanging lines), kept with its
  // plans across load steps until the mesh changes
  std::unique_ptr<Constraints> base_cache;
  i64 n_u() const { return d * V; }
  i64 n_total() const { return (d + 1) * V; }
  DevForest forest() const {
    DevForest f;
    f.d = d;
    f.n0 = n0;
    f.nroots = int(roots.size());
    f.level = t_level.p;
    f.anchor = t_anchor.p;
    f.child = t_child.p;
    f.active = t_active.p;
    f.roots = t_roots.p;
    return f;
  }
  double level_edge(int l) const { return 2.0 * K / (n0 * double(i64(1) << l)); }
  double to_physical(i64 c) const { return -K + double(c) * unit; }
  i64 extent() const { return i64(n0) * kUnit; }
};

// ---- host mesh operations (mesh.cpp)
MeshDisc* mesh_create(int d, double K, int n0);
std::unique_ptr<MeshDisc> mesh_copy(const MeshDisc& m);
void mesh_refine(MeshDisc& m, std::vector<int> ids);
void mesh_uniform_refine(MeshDisc& m, int times);
int mesh_find_cell(const MeshDisc& m, const double* x);  // smallest active id containing x, -1 outside
// active_faces (mesh.cpp:225-259): rows of (cell, axis, side, neighbour, rel), device built
std::vector<int> mesh_faces(MeshDisc& m);

// ---- constraints, assembly (fem.cpp, model.cpp)
std::unique_ptr<Constraints> mesh_build_constraints(MeshDisc& m, bool clamp, i64 n_active, const i64* dofs_dev,
                                                    const double* vals_dev);
// full = base + active phi dofs (flags already set by the caller): hanging lines drop their
// active masters, adding weight * phi_old to the inhomogeneity
void mesh_full_lines(const Constraints& base, Constraints& full);
void mesh_tables(MeshDisc& m, double mu, double lam);
// plan_cs: the constraint set the plans follow (cached by uid; the base set in the Newton step);
// c: the set of this assembly, a superset of plan_cs whose extra constraints are entry-free (the
// active phi dofs): their rows and columns drop out, their rows keep the element diagonal
void mesh_assemble_residual(MeshDisc& m, const Constraints& plan_cs, const Constraints& c, const cf_material& mat,
                            const cf_regularization& reg, const double* x, const double* pt, double* R);
std::unique_ptr<BlockSystem> mesh_assemble_jacobian(MeshDisc& m, const Constraints& plan_cs, const Constraints& c,
                                                    const cf_material& mat, const cf_regularization& reg,
                                                    const double* x, const double* pt);
void mesh_rigid_body_modes(const MeshDisc& m, const Constraints& c, double* B);
double mesh_slit_band_edge(const MeshDisc& m, const cf_material& mat);
cf_regularization mesh_resolve_regularization(const MeshDisc& m, const cf_material& mat, double band_edge);
std::vector<double> mesh_initial_crack(MeshDisc& m, const cf_material& mat, double band_half, double* band_edge);
NewtonReport mesh_newton_step(MeshDisc& m, State& st, const cf_material& mat, const cf_regularization& reg,
                              const cf_solver_options& opts);
double mesh_compute_tcv(MeshDisc& m, const double* sol);
void mesh_compute_cod(MeshDisc& m, const double* sol, const double* stations_host, int ns, double* out_host);
// adaptivity (adapt.cpp): eta per active cell (device), marked ids (host vector), transfer
void mesh_jump_estimator(MeshDisc& m, const double* sol, double* eta);
std::vector<int> mesh_mark_cells(MeshDisc& m, const double* sol, const double* eta, const cf_refinement_policy& pol);
void mesh_mask_band_eta(MeshDisc& m, const double* sol, double* eta, const cf_refinement_policy& pol);
void mesh_transfer(MeshDisc& old_m, const double* old_vec, MeshDisc& new_m, double* new_vec);

}  // namespace cfb
