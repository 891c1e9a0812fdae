// Field snapshots: the reference's native text format and legacy-VTK output (io.py:88-183), written
// by the library's host runtime.  Every float is printed "%.17g" -- byte-identical to the
// reference's "{:.17g}".format(float(v)) (correctly rounded, same exponent rules) -- so native files
// round-trip bit-exactly; rows are formatted in parallel (OpenMP) into per-chunk buffers and
// written once.  The reader parses with strtod (correctly rounded), also in parallel.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ss_common.h"

namespace {

// Formats rows [0, nrows) with fmt_row(row, buf) -> appended text; joins chunks in row order.
template <class F>
int write_rows(FILE* fh, int64_t nrows, F fmt_row) {
  const int64_t chunk = 16384;
  const int64_t nchunks = (nrows + chunk - 1) / chunk;
  std::vector<std::string> out((size_t)nchunks);
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t c = 0; c < nchunks; ++c) {
    std::string& s = out[(size_t)c];
    s.reserve((size_t)chunk * 64);
    const int64_t r1 = std::min(nrows, (c + 1) * chunk);
    for (int64_t r = c * chunk; r < r1; ++r) fmt_row(r, s);
  }
  for (const std::string& s : out)
    if (!s.empty() && fwrite(s.data(), 1, s.size(), fh) != s.size()) return 1;
  return 0;
}

inline void put_g(std::string& s, double v) {
  char b[40];
  const int n = snprintf(b, sizeof(b), "%.17g", v);
  s.append(b, (size_t)n);
}

inline void put_row(std::string& s, const double* a, int na, const double* b, int nb, int pad) {
  bool first = true;
  auto one = [&](double v) {
    if (!first) s.push_back(' ');
    first = false;
    put_g(s, v);
  };
  for (int i = 0; i < na; ++i) one(a[i]);
  for (int i = 0; i < nb; ++i) one(b[i]);
  for (int i = 0; i < pad; ++i) one(0.0);
  s.push_back('\n');
}

struct File {
  FILE* f;
  explicit File(const char* path, const char* mode) : f(fopen(path, mode)) {}
  ~File() { if (f) fclose(f); }
};

}  // namespace

// Native snapshot (io.py:104-114): header, "velocity", rows "x.. v..", "pressure", rows "p".
extern "C" int ss_write_snapshot(const char* path, int dim, int64_t n_vel, int64_t n_vert, const double* nodes,
                                 const double* velocity, const double* pressure, double time) {
  if (!path || (dim != 2 && dim != 3) || n_vel < 0 || n_vert < 0 || (n_vel && (!nodes || !velocity)) ||
      (n_vert && !pressure)) {
    ss_set_error("ss_write_snapshot: bad arguments");
    return SS_ERR_ARG;
  }
  File fh(path, "wb");
  if (!fh.f) { ss_set_error(std::string("cannot open ") + path); return SS_ERR_ARG; }
  std::string head = "snapshot " + std::to_string(dim) + " " + std::to_string(n_vel) + " " + std::to_string(n_vert) + " ";
  put_g(head, time);
  head += "\nvelocity\n";
  fwrite(head.data(), 1, head.size(), fh.f);
  if (write_rows(fh.f, n_vel, [&](int64_t r, std::string& s) {
        put_row(s, nodes + r * dim, dim, velocity + r * dim, dim, 0);
      })) { ss_set_error("write failed"); return SS_ERR_ARG; }
  fputs("pressure\n", fh.f);
  if (write_rows(fh.f, n_vert, [&](int64_t r, std::string& s) { put_row(s, pressure + r, 1, nullptr, 0, 0); })) {
    ss_set_error("write failed");
    return SS_ERR_ARG;
  }
  return SS_OK;
}

// Legacy-VTK ASCII unstructured grid with quadratic cells (io.py:129-183).  velocity / pressure may
// be null; mid-edge pressures are the averages of the edge endpoints.
extern "C" int ss_write_vtk(const char* path, const char* title, int dim, int64_t n_vel, int64_t n_vert,
                            const double* nodes, int64_t ne, int nloc, const int64_t* vel_conn, const int64_t* edges,
                            const double* velocity, const double* pressure) {
  if (!path || !title || (dim != 2 && dim != 3) || n_vel < n_vert || !nodes || (ne && !vel_conn) || nloc < 1 ||
      (pressure && n_vel > n_vert && !edges)) {
    ss_set_error("ss_write_vtk: bad arguments");
    return SS_ERR_ARG;
  }
  File fh(path, "wb");
  if (!fh.f) { ss_set_error(std::string("cannot open ") + path); return SS_ERR_ARG; }
  std::string h = std::string("# vtk DataFile Version 3.0\n") + title + "\nASCII\nDATASET UNSTRUCTURED_GRID\n" +
                  "POINTS " + std::to_string(n_vel) + " double\n";
  fwrite(h.data(), 1, h.size(), fh.f);
  int bad = write_rows(fh.f, n_vel, [&](int64_t r, std::string& s) { put_row(s, nodes + r * dim, dim, nullptr, 0, 3 - dim); });
  h = "CELLS " + std::to_string(ne) + " " + std::to_string(ne * (1 + nloc)) + "\n";
  fwrite(h.data(), 1, h.size(), fh.f);
  bad |= write_rows(fh.f, ne, [&](int64_t e, std::string& s) {
    s += std::to_string(nloc);
    for (int a = 0; a < nloc; ++a) {
      s.push_back(' ');
      s += std::to_string(vel_conn[e * nloc + a]);
    }
    s.push_back('\n');
  });
  h = "CELL_TYPES " + std::to_string(ne) + "\n";
  fwrite(h.data(), 1, h.size(), fh.f);
  const char* ct = dim == 2 ? "22\n" : "24\n";
  bad |= write_rows(fh.f, ne, [&](int64_t, std::string& s) { s += ct; });
  if (velocity || pressure) {
    h = "POINT_DATA " + std::to_string(n_vel) + "\n";
    fwrite(h.data(), 1, h.size(), fh.f);
    if (velocity) {
      fputs("VECTORS velocity double\n", fh.f);
      bad |= write_rows(fh.f, n_vel, [&](int64_t r, std::string& s) { put_row(s, velocity + r * dim, dim, nullptr, 0, 3 - dim); });
    }
    if (pressure) {
      fputs("SCALARS pressure double 1\nLOOKUP_TABLE default\n", fh.f);
      bad |= write_rows(fh.f, n_vel, [&](int64_t r, std::string& s) {
        double p;
        if (r < n_vert) {
          p = pressure[r];
        } else {
          const int64_t* ed = edges + 2 * (r - n_vert);
          p = 0.5 * (pressure[ed[0]] + pressure[ed[1]]);
        }
        put_row(s, &p, 1, nullptr, 0, 0);
      });
    }
  }
  if (bad) { ss_set_error("write failed"); return SS_ERR_ARG; }
  return SS_OK;
}

// Bulk parse of a native snapshot's two data blocks (io.py:117-134).  The caller has validated the
// header; header_lines = 2 (header + "velocity").  Returns SS_ERR_ARG with a message naming what
// is missing when the layout does not match.
extern "C" int ss_read_snapshot(const char* path, int dim, int64_t n_vel, int64_t n_vert, double* coords,
                                double* velocity, double* pressure) {
  if (!path || (dim != 2 && dim != 3) || n_vel < 0 || n_vert < 0) { ss_set_error("ss_read_snapshot: bad arguments"); return SS_ERR_ARG; }
  File fh(path, "rb");
  if (!fh.f) { ss_set_error(std::string("cannot open ") + path); return SS_ERR_ARG; }
  fseek(fh.f, 0, SEEK_END);
  const long sz = ftell(fh.f);
  fseek(fh.f, 0, SEEK_SET);
  std::vector<char> buf((size_t)sz + 1, '\0');
  if (sz > 0 && fread(buf.data(), 1, (size_t)sz, fh.f) != (size_t)sz) { ss_set_error("read failed"); return SS_ERR_ARG; }
  // line starts
  std::vector<int64_t> ls;
  ls.reserve((size_t)(n_vel + n_vert + 8));
  ls.push_back(0);
  for (long i = 0; i < sz; ++i)
    if (buf[i] == '\n') { buf[i] = '\0'; ls.push_back(i + 1); }
  const int64_t nlines = (int64_t)ls.size();
  auto line = [&](int64_t i) -> const char* { return i < nlines ? buf.data() + ls[(size_t)i] : ""; };
  auto trimmed_eq = [](const char* s, const char* w) {
    while (*s == ' ' || *s == '\t' || *s == '\r') ++s;
    const size_t n = strlen(w);
    if (strncmp(s, w, n)) return false;
    s += n;
    while (*s == ' ' || *s == '\t' || *s == '\r') ++s;
    return *s == '\0';
  };
  if (!trimmed_eq(line(1), "velocity")) { ss_set_error("missing velocity block"); return SS_ERR_ARG; }
  const int64_t p_at = 2 + n_vel;
  if (!trimmed_eq(line(p_at), "pressure")) { ss_set_error("missing pressure block"); return SS_ERR_ARG; }
  if (p_at + 1 + n_vert > nlines) { ss_set_error("truncated pressure block"); return SS_ERR_ARG; }
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
  for (int64_t r = 0; r < n_vel; ++r) {
    const char* s = line(2 + r);
    char* end;
    for (int k = 0; k < 2 * dim; ++k) {
      const double v = strtod(s, &end);
      if (end == s) { bad = 1; break; }
      if (k < dim) coords[r * dim + k] = v;
      else velocity[r * dim + k - dim] = v;
      s = end;
    }
  }
#pragma omp parallel for schedule(static) reduction(| : bad)
  for (int64_t r = 0; r < n_vert; ++r) {
    const char* s = line(p_at + 1 + r);
    char* end;
    pressure[r] = strtod(s, &end);
    if (end == s) bad = 1;
  }
  if (bad) { ss_set_error("malformed number in snapshot"); return SS_ERR_ARG; }
  return SS_OK;
}
