// FS-FEM CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.h).
//
// Written from PAPER.md (arxiv 2001.08849, juSFEM) in the paper's order and notation.
// Compiled with -O2 -ffp-contract=off: no FMA contraction, machine-independent rounding.
// Single-threaded except ora_spmv/ora_pcg row loops (each row still summed sequentially,
// dots use fixed 4096-element chunks), so results do not depend on the thread count.
//
// Readings of the paper that this file relies on are listed in DESIGN.md "Readings"
// (Q1 material matrix, Q5 P = 6/4, Q6 |det|, Q7 outward normals, Q8 BC modes, Q9 PCG,
// Q11 face order, Q12 dof = 3*node + comp, Q13 structural zeros kept).
#include "oracle.h"

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

namespace {

struct FaceRec {
  int n = 0;                    // number of (tet, opp) owners seen
  int32_t tet[3] = {-1, -1, -1};
  int32_t opp[3] = {-1, -1, -1};
};

struct Csr {
  int64_t row_lo = 0, n_rows = 0;
  std::vector<int64_t> row_ptr;
  std::vector<int32_t> col;
  std::vector<double> val;
};

}  // namespace

struct ora_mesh {
  int64_t nn = 0, nt = 0;
  std::vector<double> xyz;
  std::vector<int32_t> tets;
  // O2 output
  bool faces_built = false;
  int64_t n_interior = 0;
  std::vector<std::array<int32_t, 3>> face_nodes;
  std::vector<std::array<int32_t, 2>> face_tet, face_opp;
  // O5 output
  bool have_csr = false;
  Csr K;
  int64_t last_coo = 0;  // number of COO triplets emitted by the last assembly (Eq. 12 count)
  // O6 output
  bool have_rhs = false;
  std::vector<double> f;
  std::string err;
};

namespace {

int fail(ora_mesh* m, int code, const std::string& msg) {
  m->err = msg;
  return code;
}

struct V3 {
  double x, y, z;
};
V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
V3 cross(V3 a, V3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
double norm(V3 a) { return std::sqrt(dot(a, a)); }

V3 node(const ora_mesh* m, int64_t i) { return {m->xyz[3 * i], m->xyz[3 * i + 1], m->xyz[3 * i + 2]}; }

// 3x3 determinant by cofactor expansion along the first row.
double det3(double a11, double a12, double a13, double a21, double a22, double a23, double a31,
            double a32, double a33) {
  return a11 * (a22 * a33 - a23 * a32) - a12 * (a21 * a33 - a23 * a31) + a13 * (a21 * a32 - a22 * a31);
}

// Eq. 10: V_ABCD = (1/6) det [[xA yA zA 1]; [xB yB zB 1]; ...],
// the 4x4 determinant expanded along its last column (signed; Q6: volume = |.|).
double eq10_volume(V3 A, V3 B, V3 C, V3 D) {
  const V3 P[4] = {A, B, C, D};
  double det = 0.0;
  for (int r = 0; r < 4; ++r) {
    double m[3][3];
    int k = 0;
    for (int s = 0; s < 4; ++s) {
      if (s == r) continue;
      m[k][0] = P[s].x;
      m[k][1] = P[s].y;
      m[k][2] = P[s].z;
      ++k;
    }
    const double minor = det3(m[0][0], m[0][1], m[0][2], m[1][0], m[1][1], m[1][2], m[2][0], m[2][1], m[2][2]);
    const double sign = ((r + 3) % 2 == 0) ? 1.0 : -1.0;  // cofactor sign (-1)^(r+4) (0-based r, col 3)
    det += sign * minor;  // entry in column 4 is 1
  }
  return det / 6.0;
}

// Isotropic material matrix c (Q1), Voigt order (xx, yy, zz, yz, xz, xy), engineering shear.
void material(double E, double nu, double c[6][6]) {
  const double lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
  const double mu = E / (2.0 * (1.0 + nu));
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) c[i][j] = 0.0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) c[i][j] = lam;
  for (int i = 0; i < 3; ++i) c[i][i] = lam + 2.0 * mu;
  for (int i = 3; i < 6; ++i) c[i][i] = mu;
}

// Eq. 4 layout: the 6x3 block B_I for node I with b = (b_x, b_y, b_z).
void eq4_block(const double b[3], double B[6][3]) {
  const double bx = b[0], by = b[1], bz = b[2];
  const double rows[6][3] = {{bx, 0, 0}, {0, by, 0}, {0, 0, bz}, {0, bz, by}, {bz, 0, bx}, {by, bx, 0}};
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c < 3; ++c) B[r][c] = rows[r][c];
}

// Dense K_loc = V * B^T (c B) for n field nodes with vectors b[n][3]; K_loc is (3n)x(3n).
void dense_stiffness(int n, const double (*b)[3], double V, const double c[6][6], std::vector<double>& K) {
  const int m = 3 * n;
  std::vector<double> B(6 * m, 0.0), cB(6 * m, 0.0);
  for (int I = 0; I < n; ++I) {
    double blk[6][3];
    eq4_block(b[I], blk);
    for (int r = 0; r < 6; ++r)
      for (int a = 0; a < 3; ++a) B[r * m + 3 * I + a] = blk[r][a];
  }
  for (int r = 0; r < 6; ++r)
    for (int j = 0; j < m; ++j) {
      double s = 0.0;
      for (int k = 0; k < 6; ++k) s += c[r][k] * B[k * m + j];
      cB[r * m + j] = s;
    }
  K.assign(static_cast<size_t>(m) * m, 0.0);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) {
      double s = 0.0;
      for (int k = 0; k < 6; ++k) s += B[k * m + i] * cB[k * m + j];
      K[static_cast<size_t>(i) * m + j] = V * s;
    }
}

struct Triplet {
  int64_t row;
  int32_t col;
  double val;
};

// COO -> CSR (PAPER.md:449 sparse()): stable sort by (row, col) keeping emission order,
// duplicates summed in that order.  Implemented as a stable counting sort by row followed by
// a stable sort by column inside each row (same permutation as one stable (row,col) sort).
void coo_to_csr(const std::vector<Triplet>& coo, int64_t row_lo, int64_t n_rows, Csr& out) {
  std::vector<int64_t> cnt(n_rows + 1, 0);
  for (const auto& t : coo) cnt[t.row - row_lo + 1]++;
  for (int64_t r = 0; r < n_rows; ++r) cnt[r + 1] += cnt[r];
  std::vector<std::pair<int32_t, double>> byrow(coo.size());
  std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
  for (const auto& t : coo) byrow[pos[t.row - row_lo]++] = {t.col, t.val};
  out.row_lo = row_lo;
  out.n_rows = n_rows;
  out.row_ptr.assign(n_rows + 1, 0);
  out.col.clear();
  out.val.clear();
  for (int64_t r = 0; r < n_rows; ++r) {
    auto b = byrow.begin() + cnt[r], e = byrow.begin() + cnt[r + 1];
    std::stable_sort(b, e, [](const std::pair<int32_t, double>& x, const std::pair<int32_t, double>& y) {
      return x.first < y.first;
    });
    for (auto it = b; it != e;) {
      const int32_t c = it->first;
      double s = 0.0;
      for (; it != e && it->first == c; ++it) s += it->second;
      out.col.push_back(c);
      out.val.push_back(s);
    }
    out.row_ptr[r + 1] = static_cast<int64_t>(out.col.size());
  }
}

double bbox_diag(const ora_mesh* m) {
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = 0; i < m->nn; ++i)
    for (int a = 0; a < 3; ++a) {
      lo[a] = std::min(lo[a], m->xyz[3 * i + a]);
      hi[a] = std::max(hi[a], m->xyz[3 * i + a]);
    }
  const double dx = hi[0] - lo[0], dy = hi[1] - lo[1], dz = hi[2] - lo[2];
  return std::sqrt(dx * dx + dy * dy + dz * dz);
}

// Chunked dot product: fixed 4096-element chunks summed sequentially, chunk sums summed in order.
double cdot(const std::vector<double>& a, const std::vector<double>& b) {
  const int64_t n = static_cast<int64_t>(a.size());
  const int64_t C = 4096;
  const int64_t nc = (n + C - 1) / C;
  std::vector<double> part(nc, 0.0);
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < nc; ++k) {
    double s = 0.0;
    for (int64_t i = k * C; i < std::min(n, (k + 1) * C); ++i) s += a[i] * b[i];
    part[k] = s;
  }
  double s = 0.0;
  for (int64_t k = 0; k < nc; ++k) s += part[k];
  return s;
}

void spmv(const Csr& K, const double* x, double* y) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < K.n_rows; ++r) {
    double s = 0.0;
    for (int64_t k = K.row_ptr[r]; k < K.row_ptr[r + 1]; ++k) s += K.val[k] * x[K.col[k]];
    y[r] = s;
  }
}

// Banded Cholesky (textbook LL^T restricted to the band, which holds all fill), then solve.
int band_cholesky_solve(const std::vector<std::vector<std::pair<int32_t, double>>>& rows, int64_t n,
                        const std::vector<double>& rhs, std::vector<double>& x, std::string& err) {
  int64_t bw = 0;
  for (int64_t i = 0; i < n; ++i)
    for (const auto& e : rows[i]) bw = std::max<int64_t>(bw, i - e.first);
  const int64_t w = bw + 1;  // L(i, j) stored at A[i*w + (j - i + bw)], j in [i-bw, i]
  std::vector<double> A(static_cast<size_t>(n) * w, 0.0);
  for (int64_t i = 0; i < n; ++i)
    for (const auto& e : rows[i])
      if (e.first <= i) A[i * w + (e.first - i + bw)] += e.second;
  for (int64_t j = 0; j < n; ++j) {
    double d = A[j * w + bw];
    for (int64_t k = std::max<int64_t>(0, j - bw); k < j; ++k) {
      const double l = A[j * w + (k - j + bw)];
      d -= l * l;
    }
    if (!(d > 0.0)) {
      err = "cholesky: matrix not positive definite at row " + std::to_string(j);
      return 5;
    }
    const double ljj = std::sqrt(d);
    A[j * w + bw] = ljj;
    for (int64_t i = j + 1; i <= std::min(n - 1, j + bw); ++i) {
      double s = A[i * w + (j - i + bw)];
      for (int64_t k = std::max<int64_t>(0, i - bw); k < j; ++k) s -= A[i * w + (k - i + bw)] * A[j * w + (k - j + bw)];
      A[i * w + (j - i + bw)] = s / ljj;
    }
  }
  std::vector<double> y(n);
  for (int64_t i = 0; i < n; ++i) {
    double s = rhs[i];
    for (int64_t k = std::max<int64_t>(0, i - bw); k < i; ++k) s -= A[i * w + (k - i + bw)] * y[k];
    y[i] = s / A[i * w + bw];
  }
  x.assign(n, 0.0);
  for (int64_t i = n - 1; i >= 0; --i) {
    double s = y[i];
    for (int64_t k = i + 1; k <= std::min(n - 1, i + bw); ++k) s -= A[k * w + (i - k + bw)] * x[k];
    x[i] = s / A[i * w + bw];
  }
  return 0;
}

}  // namespace

extern "C" {

ora_mesh* ora_new(const double* xyz, int64_t nn, const int32_t* tets, int64_t nt) {
  ora_mesh* m = new ora_mesh();
  m->nn = nn;
  m->nt = nt;
  m->xyz.assign(xyz, xyz + 3 * nn);
  m->tets.assign(tets, tets + 4 * nt);
  return m;
}

void ora_free(ora_mesh* m) { delete m; }

const char* ora_error(const ora_mesh* m) { return m ? m->err.c_str() : "null handle"; }

int ora_validate(ora_mesh* m, double* vol_out) {
  if (m->nn < 4 || m->nt < 1) return fail(m, 1, "need at least 4 nodes and 1 tet");
  for (int64_t t = 0; t < m->nt; ++t)
    for (int a = 0; a < 4; ++a) {
      const int32_t v = m->tets[4 * t + a];
      if (v < 0 || v >= m->nn) return fail(m, 1, "tet " + std::to_string(t) + " has node id out of range");
      for (int b = 0; b < a; ++b)
        if (m->tets[4 * t + b] == v) return fail(m, 3, "tet " + std::to_string(t) + " repeats a node");
    }
  const double d = bbox_diag(m);
  const double tol = 1e-14 * d * d * d;  // SPEC.md:105 degenerate threshold
  for (int64_t t = 0; t < m->nt; ++t) {
    const int32_t* v = &m->tets[4 * t];
    const double V = eq10_volume(node(m, v[0]), node(m, v[1]), node(m, v[2]), node(m, v[3]));
    if (vol_out) vol_out[t] = V;
    if (std::fabs(V) <= tol) return fail(m, 3, "tet " + std::to_string(t) + " is degenerate");
  }
  return 0;
}

int ora_build_faces(ora_mesh* m, int64_t* n_faces, int64_t* n_interior) {
  // Face l of tet t is the face opposite its vertex l (Fig. 7: "remaining point").
  std::map<std::array<int32_t, 3>, FaceRec> table;
  for (int64_t t = 0; t < m->nt; ++t)
    for (int l = 0; l < 4; ++l) {
      std::array<int32_t, 3> key;
      int k = 0;
      for (int a = 0; a < 4; ++a)
        if (a != l) key[k++] = m->tets[4 * t + a];
      std::sort(key.begin(), key.end());
      FaceRec& rec = table[key];
      if (rec.n < 3) {
        rec.tet[rec.n] = static_cast<int32_t>(t);
        rec.opp[rec.n] = m->tets[4 * t + l];
      }
      rec.n++;
    }
  m->face_nodes.clear();
  m->face_tet.clear();
  m->face_opp.clear();
  m->n_interior = 0;
  for (const auto& kv : table) {
    if (kv.second.n > 2) {
      m->faces_built = false;
      return fail(m, 2, "face (" + std::to_string(kv.first[0]) + "," + std::to_string(kv.first[1]) + "," +
                            std::to_string(kv.first[2]) + ") is shared by more than two tets");
    }
    m->face_nodes.push_back(kv.first);
    if (kv.second.n == 2) {
      m->face_tet.push_back({kv.second.tet[0], kv.second.tet[1]});  // insertion order: t0 < t1
      m->face_opp.push_back({kv.second.opp[0], kv.second.opp[1]});
      m->n_interior++;
    } else {
      m->face_tet.push_back({kv.second.tet[0], -1});
      m->face_opp.push_back({kv.second.opp[0], -1});
    }
  }
  m->faces_built = true;
  *n_faces = static_cast<int64_t>(m->face_nodes.size());
  *n_interior = m->n_interior;
  return 0;
}

void ora_get_faces(const ora_mesh* m, int32_t* face_nodes, int32_t* face_tet, int32_t* face_opp) {
  for (size_t f = 0; f < m->face_nodes.size(); ++f) {
    for (int a = 0; a < 3; ++a) face_nodes[3 * f + a] = m->face_nodes[f][a];
    for (int a = 0; a < 2; ++a) {
      face_tet[2 * f + a] = m->face_tet[f][a];
      face_opp[2 * f + a] = m->face_opp[f][a];
    }
  }
}

int ora_face_domain(ora_mesh* m, int64_t f, int32_t* field, double* bbar, double* Vf, int* P, double* tri) {
  if (!m->faces_built) return fail(m, 6, "faces not built");
  if (f < 0 || f >= static_cast<int64_t>(m->face_nodes.size())) return fail(m, 1, "face id out of range");
  // Field nodes (Table 1 columns): A, B, C = face nodes a < b < c; D = opp0; E = opp1.
  const int32_t a = m->face_nodes[f][0], b = m->face_nodes[f][1], c = m->face_nodes[f][2];
  const int32_t t[2] = {m->face_tet[f][0], m->face_tet[f][1]};
  const int ntet = (t[1] >= 0) ? 2 : 1;
  const int32_t fld[5] = {a, b, c, m->face_opp[f][0], m->face_opp[f][1]};
  const int nf = 3 + ntet;
  for (int i = 0; i < 5; ++i) field[i] = fld[i];

  // A point is carried with its coordinates and its shape-function values on the field nodes.
  // Coordinates are taken relative to face node A (reading Q24: Eq. 7 does not depend on the
  // origin; a face-local origin keeps the far-from-origin tip faces accurate to ~1e-15).
  const V3 origin = node(m, a);
  auto local = [&](int32_t i) { return sub(node(m, i), origin); };
  struct Pt {
    V3 x;
    double N[5];
  };
  auto field_pt = [&](int I) {
    Pt p;
    p.x = local(fld[I]);
    for (int J = 0; J < 5; ++J) p.N[J] = (J == I) ? 1.0 : 0.0;
    return p;
  };
  // Centroid of owner tet k (points F, G of Fig. 1; row F/G of Table 1: 1/4 on its 4 nodes).
  auto centroid = [&](int k) {
    Pt p;
    const int32_t* v = &m->tets[4 * t[k]];
    V3 s = {0, 0, 0};
    for (int q = 0; q < 4; ++q) {
      const V3 x = local(v[q]);
      s.x += x.x;
      s.y += x.y;
      s.z += x.z;
    }
    p.x = {s.x / 4.0, s.y / 4.0, s.z / 4.0};
    // tet k's nodes are {A, B, C} and its remaining node (D for k = 0, E for k = 1)
    for (int J = 0; J < 5; ++J) p.N[J] = 0.0;
    p.N[0] = p.N[1] = p.N[2] = 0.25;
    p.N[3 + k] = 0.25;
    return p;
  };

  const Pt A = field_pt(0), B = field_pt(1), C = field_pt(2);
  // Boundary triangles Gamma^k (Eq. 5-7; Q5: P = 6 interior, 4 exterior), each with the
  // 4th vertex of its own sub-tetrahedron, used to orient the normal outward (Q7).
  struct Tri {
    Pt v[3];
    V3 inner;
  };
  std::vector<Tri> tris;
  double V = 0.0;
  for (int k = 0; k < ntet; ++k) {
    const Pt G = centroid(k);
    tris.push_back({{A, B, G}, C.x});
    tris.push_back({{B, C, G}, A.x});
    tris.push_back({{C, A, G}, B.x});
    V += std::fabs(eq10_volume(A.x, B.x, C.x, G.x));  // sub-tet ABCF / ABCG (Fig. 1)
  }
  if (ntet == 1) tris.push_back({{A, B, C}, centroid(0).x});
  *Vf = V;
  *P = static_cast<int>(tris.size());

  double acc[5][3] = {};
  for (size_t i = 0; i < tris.size(); ++i) {
    const Tri& T = tris[i];
    const V3 cr = cross(sub(T.v[1].x, T.v[0].x), sub(T.v[2].x, T.v[0].x));
    const double area = 0.5 * norm(cr);  // Eq. 11
    V3 n = {cr.x / norm(cr), cr.y / norm(cr), cr.z / norm(cr)};
    if (dot(n, sub(T.inner, T.v[0].x)) > 0.0) n = {-n.x, -n.y, -n.z};  // outward (Q7)
    double NG[5];
    for (int J = 0; J < 5; ++J) NG[J] = (T.v[0].N[J] + T.v[1].N[J] + T.v[2].N[J]) / 3.0;  // Table 1 g-rows
    const double nv[3] = {n.x, n.y, n.z};
    for (int I = 0; I < nf; ++I)
      for (int h = 0; h < 3; ++h) acc[I][h] += nv[h] * NG[I] * area;  // Eq. 7 summand
    if (tri) {
      double* o = tri + 9 * i;
      o[0] = area;
      o[1] = n.x;
      o[2] = n.y;
      o[3] = n.z;
      for (int J = 0; J < 5; ++J) o[4 + J] = NG[J];
    }
  }
  for (int I = 0; I < 5; ++I)
    for (int h = 0; h < 3; ++h) bbar[3 * I + h] = (I < nf) ? acc[I][h] / V : 0.0;  // Eq. 7: (1/V_k) sum
  return 0;
}

int ora_assemble_fs(ora_mesh* m, double E, double nu, int64_t node_lo, int64_t node_hi) {
  if (!m->faces_built) return fail(m, 6, "faces not built");
  if (!(E > 0.0) || !(nu > -1.0 && nu < 0.5)) return fail(m, 1, "material out of range");
  if (node_lo < 0 || node_hi > m->nn || node_lo >= node_hi) return fail(m, 1, "bad node range");
  double c[6][6];
  material(E, nu, c);
  std::vector<Triplet> coo;
  std::vector<double> Kf;
  const int64_t nf_tot = static_cast<int64_t>(m->face_nodes.size());
  for (int64_t f = 0; f < nf_tot; ++f) {
    int32_t fld[5];
    double bb[15], Vf;
    int P;
    // Faces that cannot emit a kept row are skipped before any arithmetic (row filter only).
    bool any = false;
    const int32_t cand[5] = {m->face_nodes[f][0], m->face_nodes[f][1], m->face_nodes[f][2], m->face_opp[f][0],
                             m->face_opp[f][1]};
    for (int I = 0; I < 5; ++I)
      if (cand[I] >= node_lo && cand[I] < node_hi) any = true;
    if (!any) continue;
    ora_face_domain(m, f, fld, bb, &Vf, &P, nullptr);
    const int n = (fld[4] >= 0) ? 5 : 4;
    double b[5][3];
    for (int I = 0; I < n; ++I)
      for (int h = 0; h < 3; ++h) b[I][h] = bb[3 * I + h];
    dense_stiffness(n, b, Vf, c, Kf);  // Eq. 9 summand: B^T c B V_k
    const int mm = 3 * n;
    for (int i = 0; i < mm; ++i) {
      const int64_t gi = 3 * static_cast<int64_t>(fld[i / 3]) + i % 3;
      if (fld[i / 3] < node_lo || fld[i / 3] >= node_hi) continue;
      for (int j = 0; j < mm; ++j)
        coo.push_back({gi, static_cast<int32_t>(3 * fld[j / 3] + j % 3), Kf[static_cast<size_t>(i) * mm + j]});
    }
  }
  m->last_coo = static_cast<int64_t>(coo.size());
  coo_to_csr(coo, 3 * node_lo, 3 * (node_hi - node_lo), m->K);
  m->have_csr = true;
  m->have_rhs = false;
  return 0;
}

// FEM-T4 gradients of tet t: b[I] = grad N_I, *V = |Eq. 10 volume|.
static void tet_gradients(const ora_mesh* m, int64_t t, double b[4][3], double* V) {
  const int32_t* v = &m->tets[4 * t];
  // Linear shape functions N_I = (a_I + b_I x + c_I y + d_I z): the coefficient vectors are
  // the columns of inv([[1 x y z] per node]); gradients (b_I, c_I, d_I) via cofactors.
  V3 X[4];
  for (int I = 0; I < 4; ++I) X[I] = node(m, v[I]);
  double Mx[4][4];
  for (int I = 0; I < 4; ++I) {
    Mx[I][0] = 1.0;
    Mx[I][1] = X[I].x;
    Mx[I][2] = X[I].y;
    Mx[I][3] = X[I].z;
  }
  // det(Mx) with columns (1, x, y, z) = -(Eq. 10 determinant with columns (x, y, z, 1)).
  const double V6 = -6.0 * eq10_volume(X[0], X[1], X[2], X[3]);
  for (int I = 0; I < 4; ++I)
    for (int h = 0; h < 3; ++h) {
      // inverse(Mx)[1+h][I] = cofactor(I, 1+h) / det
      double sub3[3][3];
      int r = 0;
      for (int rr = 0; rr < 4; ++rr) {
        if (rr == I) continue;
        int cc2 = 0;
        for (int cc = 0; cc < 4; ++cc) {
          if (cc == 1 + h) continue;
          sub3[r][cc2++] = Mx[rr][cc];
        }
        ++r;
      }
      const double minor = det3(sub3[0][0], sub3[0][1], sub3[0][2], sub3[1][0], sub3[1][1], sub3[1][2],
                                sub3[2][0], sub3[2][1], sub3[2][2]);
      const double sign = ((I + 1 + h) % 2 == 0) ? 1.0 : -1.0;
      b[I][h] = sign * minor / V6;
    }
  *V = std::fabs(V6) / 6.0;
}

int ora_assemble_fem(ora_mesh* m, double E, double nu, int64_t node_lo, int64_t node_hi) {
  if (!(E > 0.0) || !(nu > -1.0 && nu < 0.5)) return fail(m, 1, "material out of range");
  if (node_lo < 0 || node_hi > m->nn || node_lo >= node_hi) return fail(m, 1, "bad node range");
  double c[6][6];
  material(E, nu, c);
  std::vector<Triplet> coo;
  std::vector<double> Ke;
  for (int64_t t = 0; t < m->nt; ++t) {
    const int32_t* v = &m->tets[4 * t];
    bool any = false;
    for (int I = 0; I < 4; ++I)
      if (v[I] >= node_lo && v[I] < node_hi) any = true;
    if (!any) continue;
    double b[4][3], Ve;
    tet_gradients(m, t, b, &Ve);
    dense_stiffness(4, b, Ve, c, Ke);
    for (int i = 0; i < 12; ++i) {
      if (v[i / 3] < node_lo || v[i / 3] >= node_hi) continue;
      const int64_t gi = 3 * static_cast<int64_t>(v[i / 3]) + i % 3;
      for (int j = 0; j < 12; ++j) coo.push_back({gi, static_cast<int32_t>(3 * v[j / 3] + j % 3), Ke[i * 12 + j]});
    }
  }
  coo_to_csr(coo, 3 * node_lo, 3 * (node_hi - node_lo), m->K);
  m->have_csr = true;
  m->have_rhs = false;
  return 0;
}

// K7: one domain's dense stiffness, 15x15 with absent field positions zero.
int ora_face_stiffness(ora_mesh* m, int64_t f, double E, double nu, double* K, int32_t* field) {
  if (!(E > 0.0) || !(nu > -1.0 && nu < 0.5)) return fail(m, 1, "material out of range");
  int32_t fld[5];
  double bb[15], Vf;
  int P;
  const int st = ora_face_domain(m, f, fld, bb, &Vf, &P, nullptr);
  if (st != 0) return st;
  double c[6][6];
  material(E, nu, c);
  const int n = (fld[4] >= 0) ? 5 : 4;
  double b[5][3];
  for (int I = 0; I < n; ++I)
    for (int h = 0; h < 3; ++h) b[I][h] = bb[3 * I + h];
  std::vector<double> Kf;
  dense_stiffness(n, b, Vf, c, Kf);  // Eq. 9 summand: B^T c B V_k
  const int mm = 3 * n;
  for (int i = 0; i < 225; ++i) K[i] = 0.0;
  for (int i = 0; i < mm; ++i)
    for (int j = 0; j < mm; ++j) K[15 * i + j] = Kf[static_cast<size_t>(i) * mm + j];
  for (int I = 0; I < 5; ++I) field[I] = fld[I];
  return 0;
}

int ora_tet_stiffness(ora_mesh* m, int64_t t, double E, double nu, double* K, int32_t* field) {
  if (!(E > 0.0) || !(nu > -1.0 && nu < 0.5)) return fail(m, 1, "material out of range");
  if (t < 0 || t >= m->nt) return fail(m, 1, "tet id out of range");
  double c[6][6];
  material(E, nu, c);
  double b[4][3], Ve;
  tet_gradients(m, t, b, &Ve);
  std::vector<double> Ke;
  dense_stiffness(4, b, Ve, c, Ke);
  for (int i = 0; i < 225; ++i) K[i] = 0.0;
  for (int i = 0; i < 12; ++i)
    for (int j = 0; j < 12; ++j) K[15 * i + j] = Ke[static_cast<size_t>(i) * 12 + j];
  for (int I = 0; I < 4; ++I) field[I] = m->tets[4 * t + I];
  field[4] = -1;
  return 0;
}

int64_t ora_last_coo_count(const ora_mesh* m) { return m->last_coo; }

int ora_set_csr(ora_mesh* m, int64_t n_rows, const int64_t* row_ptr, const int32_t* col_idx, const double* vals) {
  if (n_rows != 3 * m->nn) return fail(m, 1, "set_csr needs 3*nn rows");
  m->K.row_lo = 0;
  m->K.n_rows = n_rows;
  m->K.row_ptr.assign(row_ptr, row_ptr + n_rows + 1);
  m->K.col.assign(col_idx, col_idx + row_ptr[n_rows]);
  m->K.val.assign(vals, vals + row_ptr[n_rows]);
  m->have_csr = true;
  m->have_rhs = false;
  return 0;
}

void ora_csr_dims(const ora_mesh* m, int64_t* row_lo, int64_t* n_rows, int64_t* nnz) {
  *row_lo = m->K.row_lo;
  *n_rows = m->K.n_rows;
  *nnz = m->K.row_ptr.empty() ? 0 : m->K.row_ptr.back();
}

void ora_get_csr(const ora_mesh* m, int64_t* row_ptr, int32_t* col_idx, double* vals) {
  std::memcpy(row_ptr, m->K.row_ptr.data(), sizeof(int64_t) * m->K.row_ptr.size());
  std::memcpy(col_idx, m->K.col.data(), sizeof(int32_t) * m->K.col.size());
  std::memcpy(vals, m->K.val.data(), sizeof(double) * m->K.val.size());
}

int ora_spmv(const ora_mesh* m, const double* x, double* y) {
  if (!m->have_csr || m->K.row_lo != 0 || m->K.n_rows != 3 * m->nn) return 6;
  spmv(m->K, x, y);
  return 0;
}

int ora_apply_bc(ora_mesh* m, const int32_t* dirichlet, int64_t n_dir, const double* loads, int mode,
                 double penalty_scale) {
  if (!m->have_csr || m->K.row_lo != 0 || m->K.n_rows != 3 * m->nn) return fail(m, 6, "need the full K");
  if (mode != 0 && mode != 1) return fail(m, 1, "mode must be 0 (modify) or 1 (penalty)");
  const int64_t n = 3 * m->nn;
  std::vector<char> fixed(n, 0);
  for (int64_t k = 0; k < n_dir; ++k) {
    if (dirichlet[k] < 0 || dirichlet[k] >= m->nn) return fail(m, 1, "dirichlet node out of range");
    for (int a = 0; a < 3; ++a) fixed[3 * static_cast<int64_t>(dirichlet[k]) + a] = 1;
  }
  m->f.assign(loads, loads + n);
  const std::vector<double> g(n, 0.0);  // clamped: prescribed displacement g = 0
  Csr& K = m->K;
  if (mode == 0) {
    // f_j -= K_jr g_r for free rows j (zero here since g = 0), then zero row/col r, keep K_rr.
    for (int64_t j = 0; j < n; ++j)
      for (int64_t k = K.row_ptr[j]; k < K.row_ptr[j + 1]; ++k)
        if (fixed[K.col[k]] && !fixed[j]) m->f[j] -= K.val[k] * g[K.col[k]];
    for (int64_t j = 0; j < n; ++j)
      for (int64_t k = K.row_ptr[j]; k < K.row_ptr[j + 1]; ++k)
        if ((fixed[j] || fixed[K.col[k]]) && K.col[k] != j) K.val[k] = 0.0;
    for (int64_t r = 0; r < n; ++r)
      if (fixed[r])
        for (int64_t k = K.row_ptr[r]; k < K.row_ptr[r + 1]; ++k)
          if (K.col[k] == r) m->f[r] = K.val[k] * g[r];
  } else {
    double dmax = 0.0;
    for (int64_t r = 0; r < n; ++r)
      for (int64_t k = K.row_ptr[r]; k < K.row_ptr[r + 1]; ++k)
        if (K.col[k] == r) dmax = std::max(dmax, K.val[k]);
    const double alpha = ((penalty_scale > 0.0) ? penalty_scale : 1e8) * dmax;
    for (int64_t r = 0; r < n; ++r)
      if (fixed[r])
        for (int64_t k = K.row_ptr[r]; k < K.row_ptr[r + 1]; ++k)
          if (K.col[k] == r) {
            K.val[k] += alpha;
            m->f[r] += alpha * g[r];
          }
  }
  m->have_rhs = true;
  return 0;
}

void ora_get_rhs(const ora_mesh* m, double* f) { std::memcpy(f, m->f.data(), sizeof(double) * m->f.size()); }

int ora_pcg(ora_mesh* m, double tol, int64_t max_iter, double* u, int64_t* iters, double* rel_res,
            double* true_rel_res) {
  if (!m->have_rhs) return fail(m, 6, "apply_bc first");
  const int64_t n = 3 * m->nn;
  if (tol <= 0.0) tol = 1e-10;
  if (max_iter <= 0) max_iter = std::max<int64_t>(1000, static_cast<int64_t>(20.0 * std::sqrt(static_cast<double>(n))));
  const Csr& K = m->K;
  std::vector<double> dinv(n);
  for (int64_t r = 0; r < n; ++r) {
    double d = 0.0;
    for (int64_t k = K.row_ptr[r]; k < K.row_ptr[r + 1]; ++k)
      if (K.col[k] == r) d = K.val[k];
    if (!(d > 0.0)) return fail(m, 5, "non-positive diagonal");
    dinv[r] = 1.0 / d;
  }
  std::vector<double> x(n, 0.0), r(m->f), z(n), p(n), q(n);
  const double fnorm = std::sqrt(cdot(m->f, m->f));
  int64_t it = 0;
  double rr = cdot(r, r);
  int status = 0;
  if (fnorm == 0.0) {
    rr = 0.0;
  } else if (std::sqrt(rr) > tol * fnorm) {
    for (int64_t i = 0; i < n; ++i) z[i] = dinv[i] * r[i];
    p = z;
    double rho = cdot(r, z);
    status = 4;
    while (it < max_iter) {
      spmv(K, p.data(), q.data());
      const double pq = cdot(p, q);
      if (!(pq > 0.0) || !std::isfinite(pq)) {
        status = 5;
        m->err = "pcg breakdown: p.q <= 0";
        break;
      }
      const double alpha = rho / pq;
      for (int64_t i = 0; i < n; ++i) {
        x[i] += alpha * p[i];
        r[i] -= alpha * q[i];
      }
      ++it;
      rr = cdot(r, r);
      if (std::sqrt(rr) <= tol * fnorm) {
        status = 0;
        break;
      }
      for (int64_t i = 0; i < n; ++i) z[i] = dinv[i] * r[i];
      const double rho_new = cdot(r, z);
      const double beta = rho_new / rho;
      rho = rho_new;
      for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    }
    if (status == 4) m->err = "pcg: max_iter reached";
  }
  std::memcpy(u, x.data(), sizeof(double) * n);
  *iters = it;
  *rel_res = (fnorm > 0.0) ? std::sqrt(rr) / fnorm : 0.0;
  spmv(K, x.data(), q.data());
  for (int64_t i = 0; i < n; ++i) q[i] = m->f[i] - q[i];
  *true_rel_res = (fnorm > 0.0) ? std::sqrt(cdot(q, q)) / fnorm : 0.0;
  return status;
}

int ora_cholesky(ora_mesh* m, double* u) {
  if (!m->have_rhs) return fail(m, 6, "apply_bc first");
  const int64_t n = 3 * m->nn;
  std::vector<std::vector<std::pair<int32_t, double>>> rows(n);
  for (int64_t r = 0; r < n; ++r)
    for (int64_t k = m->K.row_ptr[r]; k < m->K.row_ptr[r + 1]; ++k) rows[r].push_back({m->K.col[k], m->K.val[k]});
  std::vector<double> x;
  const int st = band_cholesky_solve(rows, n, m->f, x, m->err);
  if (st) return st;
  std::memcpy(u, x.data(), sizeof(double) * n);
  return 0;
}

int ora_cholesky_eliminate(ora_mesh* m, const int32_t* dirichlet, int64_t n_dir, const double* loads, double* u) {
  if (!m->have_csr || m->K.row_lo != 0 || m->K.n_rows != 3 * m->nn) return fail(m, 6, "need the full K");
  const int64_t n = 3 * m->nn;
  std::vector<char> fixed(n, 0);
  for (int64_t k = 0; k < n_dir; ++k)
    for (int a = 0; a < 3; ++a) fixed[3 * static_cast<int64_t>(dirichlet[k]) + a] = 1;
  std::vector<int64_t> red(n, -1);  // reduced index of each free dof
  int64_t nr = 0;
  for (int64_t i = 0; i < n; ++i)
    if (!fixed[i]) red[i] = nr++;
  std::vector<std::vector<std::pair<int32_t, double>>> rows(nr);
  std::vector<double> rhs(nr);
  for (int64_t i = 0; i < n; ++i) {
    if (fixed[i]) continue;
    rhs[red[i]] = loads[i];
    for (int64_t k = m->K.row_ptr[i]; k < m->K.row_ptr[i + 1]; ++k)
      if (!fixed[m->K.col[k]]) rows[red[i]].push_back({static_cast<int32_t>(red[m->K.col[k]]), m->K.val[k]});
  }
  std::vector<double> x;
  const int st = band_cholesky_solve(rows, nr, rhs, x, m->err);
  if (st) return st;
  for (int64_t i = 0; i < n; ++i) u[i] = fixed[i] ? 0.0 : x[red[i]];
  return 0;
}

}  // extern "C"

// O9 ("first obtain the nodal displacements and then the strain
// and stress", 457): per smoothing domain k the smoothed strain of Eq. 2 with the B-bar of Eq. 4,
// eps_k = B_k d_k (Voigt xx, yy, zz, yz, xz, xy, engineering shear), sigma_k = c eps_k; per node
// the volume-weighted mean over the domains whose field holds the node (averaging rule: reading
// Q27, the paper does not state one), and the von Mises stress of that mean.
int ora_recover(ora_mesh* m, double E, double nu, const double* u, double* strain, double* stress,
                double* node_stress, double* node_vm) {
  if (!m->faces_built) return fail(m, 6, "faces not built");
  double c[6][6];
  material(E, nu, c);
  const int64_t nf = static_cast<int64_t>(m->face_nodes.size());
  std::vector<double> acc(6 * static_cast<size_t>(m->nn), 0.0), w(static_cast<size_t>(m->nn), 0.0);
  for (int64_t f = 0; f < nf; ++f) {
    int32_t fld[5];
    double bb[15], Vf;
    int P;
    ora_face_domain(m, f, fld, bb, &Vf, &P, nullptr);
    const int n = (fld[4] >= 0) ? 5 : 4;
    double eps[6] = {0, 0, 0, 0, 0, 0};
    for (int I = 0; I < n; ++I) {
      double blk[6][3];
      eq4_block(&bb[3 * I], blk);  // Eq. 4 block of node I
      for (int r = 0; r < 6; ++r)
        for (int a = 0; a < 3; ++a) eps[r] += blk[r][a] * u[3 * static_cast<int64_t>(fld[I]) + a];
    }
    double sig[6];
    for (int r = 0; r < 6; ++r) {
      double s = 0.0;
      for (int k = 0; k < 6; ++k) s += c[r][k] * eps[k];
      sig[r] = s;
    }
    for (int r = 0; r < 6; ++r) {
      if (strain) strain[6 * f + r] = eps[r];
      if (stress) stress[6 * f + r] = sig[r];
    }
    for (int I = 0; I < n; ++I) {
      for (int r = 0; r < 6; ++r) acc[6 * static_cast<size_t>(fld[I]) + r] += Vf * sig[r];
      w[fld[I]] += Vf;
    }
  }
  for (int64_t i = 0; i < m->nn; ++i) {
    double s[6];
    for (int r = 0; r < 6; ++r) s[r] = (w[i] > 0.0) ? acc[6 * i + r] / w[i] : 0.0;
    if (node_stress)
      for (int r = 0; r < 6; ++r) node_stress[6 * i + r] = s[r];
    if (node_vm) {
      const double d01 = s[0] - s[1], d12 = s[1] - s[2], d20 = s[2] - s[0];
      node_vm[i] = std::sqrt(0.5 * (d01 * d01 + d12 * d12 + d20 * d20) + 3.0 * (s[3] * s[3] + s[4] * s[4] + s[5] * s[5]));
    }
  }
  return 0;
}

// O10 ("the nodal load is calculated"; 496-499 §4.1: uniform pressure on the upper
// face): a uniform traction t on the exterior faces whose three nodes are all
// flagged gives each of those nodes t * A / 3 (A from Eq. 11), accumulated in face order.
int ora_surface_loads(ora_mesh* m, const uint8_t* node_flag, const double* traction, double* loads) {
  if (!m->faces_built) return fail(m, 6, "faces not built");
  for (int64_t i = 0; i < 3 * m->nn; ++i) loads[i] = 0.0;
  const int64_t nf = static_cast<int64_t>(m->face_nodes.size());
  for (int64_t f = 0; f < nf; ++f) {
    if (m->face_tet[f][1] >= 0) continue;  // interior face
    const int32_t* v = m->face_nodes[f].data();
    if (!node_flag[v[0]] || !node_flag[v[1]] || !node_flag[v[2]]) continue;
    const V3 a = node(m, v[0]), b = node(m, v[1]), c = node(m, v[2]);
    const double area = 0.5 * norm(cross(sub(b, a), sub(c, a)));  // Eq. 11
    for (int k = 0; k < 3; ++k)
      for (int h = 0; h < 3; ++h) loads[3 * static_cast<int64_t>(v[k]) + h] += traction[h] * area / 3.0;
  }
  return 0;
}
