// §8f row 4: I/O of device data in the reference's formats.
//
//   write_matrix_market  linsolve.cpp:478-490  "%%MatrixMarket matrix coordinate real general",
//                        1-based "i j %.17g" lines in row order (byte-identical text)
//   write_vtk            postproc.cpp:111-167  legacy VTK unstructured grid: points, cells in the
//                        reference's active-cell order (root-lexicographic, then hierarchical
//                        z-order) with the VTK corner permutation, u / phi (/ phi_old) point data;
//                        ASCII is byte-identical to the reference, BINARY is the same dataset in
//                        the legacy big-endian binary encoding (a 68M-dof solution is ~2 GB of text)
//
// The device arrays are copied to the host once; text formatting runs on all host threads in
// row / vertex chunks and the chunks are written in order.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <thread>
#include <vector>

#include "cf_vec.hpp"

namespace cfb {

namespace {

template <class T>
std::vector<T> to_host(const T* dev, i64 n) {
  std::vector<T> h(size_t(std::max<i64>(n, 0)));
  if (n > 0) {
    CF_CUDA(cudaMemcpyAsync(h.data(), dev, size_t(n) * sizeof(T), cudaMemcpyDefault, stream()));
    CF_CUDA(cudaStreamSynchronize(stream()));
  }
  return h;
}

// format items [0, n) with fn(i, out) into per-thread strings, written in order
template <class F>
void parallel_text(std::ofstream& out, i64 n, F fn) {
  const int nt = int(std::max(1u, std::min(64u, std::thread::hardware_concurrency())));
  const i64 chunk = std::max<i64>(1, (n + nt - 1) / nt);
  std::vector<std::string> parts(static_cast<size_t>(nt));
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      const i64 lo = t * chunk, hi = std::min(n, lo + chunk);
      std::string& s = parts[size_t(t)];
      for (i64 i = lo; i < hi; ++i) fn(i, s);
    });
  for (auto& x : th) x.join();
  for (auto& s : parts) out.write(s.data(), std::streamsize(s.size()));
}

void put17(std::string& s, double v) {
  char buf[40];
  const int k = std::snprintf(buf, sizeof(buf), "%.17g", v);
  s.append(buf, size_t(k));
}

// the reference's active-cell order after uniform_refine (mesh.cpp:147-169, 209-215):
// root cells lexicographic, then the 2^(d r) children in hierarchical z-order
std::vector<i64> cells_in_reference_order(const GridDesc& g) {
  std::vector<i64> order(size_t(g.ncells));
  const i64 nroot = (g.d == 3) ? i64(g.n0) * g.n0 * g.n0 : i64(g.n0) * g.n0;
  const i64 nsub = i64(1) << (g.d * g.r);
  i64 t = 0;
  for (i64 root = 0; root < nroot; ++root) {
    const i64 rx = root % g.n0, ry = (root / g.n0) % g.n0, rz = (g.d == 3) ? root / (i64(g.n0) * g.n0) : 0;
    for (i64 m = 0; m < nsub; ++m) {
      i64 l[3] = {0, 0, 0};
      for (int j = 0; j < g.r; ++j)
        for (int a = 0; a < g.d; ++a) l[a] |= ((m >> (g.d * j + a)) & 1) << j;
      const i64 cx = (rx << g.r) | l[0], cy = (ry << g.r) | l[1], cz = (rz << g.r) | l[2];
      order[size_t(t++)] = cx + g.nc * (cy + g.nc * cz);
    }
  }
  return order;
}

inline void put_be64(std::string& s, double v) {
  unsigned char b[8];
  std::memcpy(b, &v, 8);
  for (int i = 7; i >= 0; --i) s.push_back(char(b[i]));
}
inline void put_be32(std::string& s, std::int32_t v) {
  unsigned char b[4];
  std::memcpy(b, &v, 4);
  for (int i = 3; i >= 0; --i) s.push_back(char(b[i]));
}

}  // namespace

void write_matrix_market(const Csr& A, const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) fail(CF_ERR_INVALID_ARGUMENT, "write_matrix_market: cannot open " + path);
  const auto ptr = to_host(A.ptr.p, A.rows + 1);
  const auto col = to_host(A.col.p, A.nnz);
  const auto val = to_host(A.val.p, A.nnz);
  out << "%%MatrixMarket matrix coordinate real general\n";
  out << A.rows << " " << A.cols << " " << A.nnz << "\n";
  parallel_text(out, A.rows, [&](i64 i, std::string& s) {
    char buf[64];
    for (i64 k = ptr[size_t(i)]; k < ptr[size_t(i) + 1]; ++k) {
      const int n = std::snprintf(buf, sizeof(buf), "%d %d %.17g\n", int(i + 1), col[size_t(k)] + 1, val[size_t(k)]);
      s.append(buf, size_t(n));
    }
  });
  if (!out) fail(CF_ERR_NUMERICAL, "write_matrix_market: write failed for " + path);
}

void write_vtk(const Problem& P, const double* sol_dev, const double* phi_old_dev, const std::string& path,
               bool binary) {
  const GridDesc& g = P.g;
  std::ofstream out(path, std::ios::binary);
  if (!out) fail(CF_ERR_INVALID_ARGUMENT, "write_vtk: cannot open " + path);
  const auto sol = to_host(sol_dev, g.n_total());
  std::vector<double> po;
  if (phi_old_dev) po = to_host(phi_old_dev, g.V);
  const i64 nv = g.V, d = g.d, npc = i64(1) << d;
  auto coord = [&](i64 i) { return -g.K + double(i * (i64(1) << (16 - g.r))) * g.unit; };  // mesh.hpp:73-75
  out << "# vtk DataFile Version 3.0\n";
  out << "crackfield phase-field fracture\n";
  out << (binary ? "BINARY\n" : "ASCII\n");
  out << "DATASET UNSTRUCTURED_GRID\n";
  out << "POINTS " << nv << " double\n";
  parallel_text(out, nv, [&](i64 v, std::string& s) {
    const double x[3] = {coord(v % g.nn), coord((v / g.nn) % g.nn), d == 3 ? coord(v / (g.nn * g.nn)) : 0.0};
    if (binary) {
      for (double c : x) put_be64(s, c);
    } else {
      put17(s, x[0]);
      s.push_back(' ');
      put17(s, x[1]);
      s.push_back(' ');
      put17(s, x[2]);
      s.push_back('\n');
    }
  });
  if (binary) out << "\n";
  const auto order = cells_in_reference_order(g);
  static const int quad_order[4] = {0, 1, 3, 2};
  static const int hex_order[8] = {0, 1, 3, 2, 4, 5, 7, 6};
  out << "CELLS " << g.ncells << " " << g.ncells * (npc + 1) << "\n";
  parallel_text(out, g.ncells, [&](i64 t, std::string& s) {
    const i64 c = order[size_t(t)];
    const i64 cx = c % g.nc, cy = (c / g.nc) % g.nc, cz = (d == 3) ? c / (g.nc * g.nc) : 0;
    if (binary) put_be32(s, std::int32_t(npc));
    else s += std::to_string(npc);
    for (int k = 0; k < npc; ++k) {
      const int corner = (d == 2) ? quad_order[k] : hex_order[k];
      const i64 v = (cx + (corner & 1)) + g.nn * ((cy + ((corner >> 1) & 1)) + g.nn * (cz + ((corner >> 2) & 1)));
      if (binary) {
        put_be32(s, std::int32_t(v));
      } else {
        s.push_back(' ');
        s += std::to_string(v);
      }
    }
    if (!binary) s.push_back('\n');
  });
  if (binary) out << "\n";
  out << "CELL_TYPES " << g.ncells << "\n";
  parallel_text(out, g.ncells, [&](i64, std::string& s) {
    if (binary) put_be32(s, d == 2 ? 9 : 12);
    else s += (d == 2 ? "9\n" : "12\n");
  });
  if (binary) out << "\n";
  out << "POINT_DATA " << nv << "\n";
  out << "VECTORS u double\n";
  const i64 nu = g.n_u();
  parallel_text(out, nv, [&](i64 v, std::string& s) {
    const double u[3] = {sol[size_t(v * d)], sol[size_t(v * d + 1)], d == 3 ? sol[size_t(v * d + 2)] : 0.0};
    if (binary) {
      for (double c : u) put_be64(s, c);
    } else {
      put17(s, u[0]);
      s.push_back(' ');
      put17(s, u[1]);
      s.push_back(' ');
      put17(s, u[2]);
      s.push_back('\n');
    }
  });
  if (binary) out << "\n";
  auto scalars = [&](const char* name, const double* a) {
    out << "SCALARS " << name << " double 1\n";
    out << "LOOKUP_TABLE default\n";
    parallel_text(out, nv, [&](i64 v, std::string& s) {
      if (binary) {
        put_be64(s, a[v]);
      } else {
        put17(s, a[v]);
        s.push_back('\n');
      }
    });
    if (binary) out << "\n";
  };
  scalars("phi", sol.data() + nu);
  if (phi_old_dev) scalars("phi_old", po.data());
  if (!out) fail(CF_ERR_NUMERICAL, "write_vtk: write failed for " + path);
}

}  // namespace cfb
