/* tetmf_oracle.c -- plain-C restatement of the reference's CPU apply path.
 *
 * TEST INFRASTRUCTURE ONLY. This is the oracle ("port") the parity tests use
 * next to the compiled reference (oracle/_ref); it is never linked into or
 * called by the product library. Each function cites the reference code it
 * restates (paths relative to /root/reference/proj/src). Parity pinning:
 * tests/test_oracle.py checks this port against the reference itself (run
 * here through oracle/_ref and through the committed tests/golden fixtures).
 *
 * Restated algorithm:
 *   MacroMesh (mesh.cpp:76-181), micro geometry (mesh.cpp:22-74, 183-271),
 *   quadrature rules (quadrature.cpp:19-147), bases (fespace.cpp:14-113),
 *   DoFIndexer numbering + slot maps + signs (fespace.cpp:151-430),
 *   interpolate (fespace.cpp:494-506), StarTables (forms.cpp:69-131),
 *   FormSystem::apply / reference_apply (forms.cpp:195-260),
 *   config-2 harness P1 -div(k grad).
 */
#define _POSIX_C_SOURCE 199309L
#include "tetmf_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

typedef int64_t i64;

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

static _Thread_local char g_err[512];
static void set_err(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
const char* port_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ mesh */
typedef struct {
  int nv, nt;
  double (*v)[3];
  int (*t)[4];
} Mesh;

static double vol6(const Mesh* m, const int* t) { /* tet_volume6 mesh.cpp:40-44 */
  double a[3][3];
  for (int c = 0; c < 3; ++c)
    for (int r = 0; r < 3; ++r) a[r][c] = m->v[t[c + 1]][r] - m->v[t[0]][r];
  return a[0][0] * (a[1][1] * a[2][2] - a[2][1] * a[1][2]) - a[1][0] * (a[0][1] * a[2][2] - a[2][1] * a[0][2]) +
         a[2][0] * (a[0][1] * a[1][2] - a[1][1] * a[0][2]);
}

static void mesh_free(Mesh* m) {
  free(m->v);
  free(m->t);
  m->v = NULL;
  m->t = NULL;
}

static int cmp_int3(const void* a, const void* b) {
  const int* x = a;
  const int* y = b;
  for (int i = 0; i < 3; ++i)
    if (x[i] != y[i]) return x[i] < y[i] ? -1 : 1;
  return 0;
}

static void face_of(const int* t, int f, int out[3]) {
  int k = 0;
  for (int i = 0; i < 4; ++i)
    if (i != f) out[k++] = t[i];
  for (int i = 0; i < 3; ++i) /* sort 3 */
    for (int j = i + 1; j < 3; ++j)
      if (out[j] < out[i]) { int s = out[i]; out[i] = out[j]; out[j] = s; }
}

/* face multiplicities: cnt[m*4+f] = number of tets sharing face f of m */
static int* face_counts(const Mesh* m) {
  int* faces = malloc(sizeof(int) * 5 * 4 * (size_t)m->nt);
  for (int i = 0; i < m->nt; ++i)
    for (int f = 0; f < 4; ++f) {
      int* r = faces + 5 * (4 * i + f);
      face_of(m->t[i], f, r);
      r[3] = i;
      r[4] = f;
    }
  qsort(faces, 4 * (size_t)m->nt, 5 * sizeof(int), cmp_int3);
  int* cnt = calloc(4 * (size_t)m->nt, sizeof(int));
  for (size_t i = 0; i < 4 * (size_t)m->nt;) {
    size_t j = i;
    while (j < 4 * (size_t)m->nt && cmp_int3(faces + 5 * j, faces + 5 * i) == 0) ++j;
    for (size_t k = i; k < j; ++k) cnt[faces[5 * k + 3] * 4 + faces[5 * k + 4]] = (int)(j - i);
    i = j;
  }
  free(faces);
  return cnt;
}

static int mesh_validate(const Mesh* m) { /* MacroMesh::validate mesh.cpp:76-94 */
  for (int i = 0; i < m->nt; ++i) {
    for (int k = 0; k < 4; ++k)
      if (m->t[i][k] < 0 || m->t[i][k] >= m->nv) { set_err("mesh: vertex id out of range"); return 1; }
    if (vol6(m, m->t[i]) <= 0.0) { set_err("mesh: tet with non-positive volume"); return 1; }
  }
  int* cnt = face_counts(m);
  for (int i = 0; i < 4 * m->nt; ++i)
    if (cnt[i] > 2) { free(cnt); set_err("mesh: face shared by more than two tets"); return 1; }
  free(cnt);
  return 0;
}

/* K^3 Kuhn cubes with cube6's per-cube rule (mesh.cpp:122-141) */
static int mesh_kuhn(Mesh* m, int kx, int ky, int kz) {
  m->nv = (kx + 1) * (ky + 1) * (kz + 1);
  m->nt = 6 * kx * ky * kz;
  m->v = malloc(sizeof(double[3]) * m->nv);
  m->t = malloc(sizeof(int[4]) * m->nt);
  int k = 0;
  for (int z = 0; z <= kz; ++z)
    for (int y = 0; y <= ky; ++y)
      for (int x = 0; x <= kx; ++x) {
        m->v[k][0] = x; m->v[k][1] = y; m->v[k][2] = z;
        ++k;
      }
#define VID(x, y, z) ((x) + (kx + 1) * ((y) + (ky + 1) * (z)))
  static const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  int ti = 0;
  for (int cz = 0; cz < kz; ++cz)
    for (int cy = 0; cy < ky; ++cy)
      for (int cx = 0; cx < kx; ++cx)
        for (int p = 0; p < 6; ++p) {
          int a[3] = {0, 0, 0};
          a[perms[p][0]] = 1;
          int b[3] = {a[0], a[1], a[2]};
          b[perms[p][1]] = 1;
          int* t = m->t[ti++];
          t[0] = VID(cx, cy, cz);
          t[1] = VID(cx + a[0], cy + a[1], cz + a[2]);
          t[2] = VID(cx + b[0], cy + b[1], cz + b[2]);
          t[3] = VID(cx + 1, cy + 1, cz + 1);
          if (vol6(m, t) < 0.0) { int s = t[2]; t[2] = t[3]; t[3] = s; }
        }
#undef VID
  return mesh_validate(m);
}

static int mesh_load(Mesh* m, const char* path) { /* MacroMesh::load mesh.cpp:143-169 */
  FILE* f = fopen(path, "r");
  if (!f) { set_err("mesh file: cannot open %s", path); return 1; }
  int capv = 64, capt = 64;
  m->v = malloc(sizeof(double[3]) * capv);
  m->t = malloc(sizeof(int[4]) * capt);
  m->nv = m->nt = 0;
  char line[512];
  int lineno = 0;
  while (fgets(line, sizeof line, f)) {
    ++lineno;
    char tag[16];
    if (sscanf(line, "%15s", tag) != 1 || tag[0] == '#') continue;
    if (!strcmp(tag, "v")) {
      if (m->nv == capv) m->v = realloc(m->v, sizeof(double[3]) * (capv *= 2));
      if (sscanf(line, "%*s %lf %lf %lf", &m->v[m->nv][0], &m->v[m->nv][1], &m->v[m->nv][2]) != 3) {
        fclose(f); set_err("mesh file: bad vertex at line %d", lineno); return 1;
      }
      ++m->nv;
    } else if (!strcmp(tag, "t")) {
      if (m->nt == capt) m->t = realloc(m->t, sizeof(int[4]) * (capt *= 2));
      int* t = m->t[m->nt];
      if (sscanf(line, "%*s %d %d %d %d", &t[0], &t[1], &t[2], &t[3]) != 4) {
        fclose(f); set_err("mesh file: bad tet at line %d", lineno); return 1;
      }
      ++m->nt;
    } else {
      fclose(f); set_err("mesh file: unknown tag '%s' at line %d", tag, lineno); return 1;
    }
  }
  fclose(f);
  return mesh_validate(m);
}

static int mesh_by_name(Mesh* m, const char* name) { /* mesh_by_name mesh.cpp:177-181 */
  memset(m, 0, sizeof(*m));
  if (!strcmp(name, "single-tet")) {
    m->nv = 4; m->nt = 1;
    m->v = calloc(4, sizeof(double[3]));
    m->t = malloc(sizeof(int[4]));
    m->v[1][0] = 1; m->v[2][1] = 1; m->v[3][2] = 1;
    for (int i = 0; i < 4; ++i) m->t[0][i] = i;
    return mesh_validate(m);
  }
  if (!strcmp(name, "cube6")) return mesh_kuhn(m, 1, 1, 1);
  int kx, ky, kz;
  if (!strncmp(name, "cubes", 5)) {
    if (sscanf(name + 5, "%dx%dx%d", &kx, &ky, &kz) == 3) return mesh_kuhn(m, kx, ky, kz);
    if (sscanf(name + 5, "%d", &kx) == 1 && strspn(name + 5, "0123456789") == strlen(name + 5))
      return mesh_kuhn(m, kx, kx, kx);
  }
  return mesh_load(m, name);
}

/* ------------------------------------------------- micro geometry (mesh.cpp) */
static const int kOffsets[6][4][3] = {/* mesh.cpp:22-29: WU WD BU BD GU GD */
                                      {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}},
                                      {{1, 1, 0}, {0, 1, 1}, {1, 0, 1}, {1, 1, 1}},
                                      {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {1, 1, 0}},
                                      {{0, 1, 0}, {0, 0, 1}, {1, 1, 0}, {0, 1, 1}},
                                      {{1, 0, 0}, {0, 0, 1}, {1, 1, 0}, {1, 0, 1}},
                                      {{0, 0, 1}, {1, 1, 0}, {0, 1, 1}, {1, 0, 1}}};
static const int kLocalEdges[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
static const int kEdgeDirs[7][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {1, -1, 0},
                                    {1, 0, -1}, {0, 1, -1}, {1, 1, -1}};

static int loop_bound(int o, int n) { /* mesh.cpp:66-74 */
  int b = o == 0 ? n : (o == 1 ? n - 2 : n - 1);
  return b > 0 ? b : 0;
}

static int orientation_det(int o) { /* offsets_det mesh.cpp:31-38 */
  int a[3][3];
  for (int c = 0; c < 3; ++c)
    for (int r = 0; r < 3; ++r) a[r][c] = kOffsets[o][c + 1][r] - kOffsets[o][0][r];
  return a[0][0] * (a[1][1] * a[2][2] - a[1][2] * a[2][1]) - a[0][1] * (a[1][0] * a[2][2] - a[1][2] * a[2][0]) +
         a[0][2] * (a[1][0] * a[2][1] - a[1][1] * a[2][0]);
}

static int edge_class(const int d[3], int* flipped) { /* fespace.cpp:60-70 */
  int e[3] = {d[0], d[1], d[2]};
  *flipped = 0;
  if (e[0] < 0 || (e[0] == 0 && e[1] < 0) || (e[0] == 0 && e[1] == 0 && e[2] < 0)) {
    e[0] = -e[0]; e[1] = -e[1]; e[2] = -e[2];
    *flipped = 1;
  }
  for (int c = 0; c < 7; ++c)
    if (e[0] == kEdgeDirs[c][0] && e[1] == kEdgeDirs[c][1] && e[2] == kEdgeDirs[c][2]) return c;
  return -1;
}

static double det3(double a[3][3]) {
  return a[0][0] * (a[1][1] * a[2][2] - a[2][1] * a[1][2]) - a[1][0] * (a[0][1] * a[2][2] - a[2][1] * a[0][2]) +
         a[2][0] * (a[0][1] * a[1][2] - a[1][1] * a[0][2]);
}

/* micro_jacobian mesh.cpp:243-262: J = (A * D) * h, det = detA * detD * h^3 */
static void micro_jacobian(const Mesh* m, int macro, int level, int o, double J[3][3], double* det) {
  const int* t = m->t[macro];
  double A[3][3], D[3][3];
  for (int c = 0; c < 3; ++c)
    for (int r = 0; r < 3; ++r) {
      A[r][c] = m->v[t[c + 1]][r] - m->v[t[0]][r];
      D[r][c] = (double)(kOffsets[o][c + 1][r] - kOffsets[o][0][r]);
    }
  const double h = 1.0 / (double)(1 << level);
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      double s = 0.0;
      for (int k = 0; k < 3; ++k) s += A[r][k] * D[k][c];
      J[r][c] = s * h;
    }
  *det = det3(A) * (double)orientation_det(o) * h * h * h;
}

static void inverse_transpose(double J[3][3], double out[3][3]) {
  double adj[3][3];
  adj[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
  adj[0][1] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
  adj[0][2] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
  adj[1][0] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
  adj[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
  adj[1][2] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
  adj[2][0] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
  adj[2][1] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
  adj[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
  const double d = J[0][0] * adj[0][0] + J[0][1] * adj[1][0] + J[0][2] * adj[2][0];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) out[r][c] = adj[c][r] * (1.0 / d);
}

/* lattice_to_world mesh.cpp:264-271 */
static void lattice_to_world(const Mesh* m, int macro, int level, const int p[3], double out[3]) {
  const int* t = m->t[macro];
  const double h = 1.0 / (double)(1 << level);
  for (int r = 0; r < 3; ++r) {
    const double p0 = m->v[t[0]][r];
    out[r] = p0 + h * (((double)p[0] * (m->v[t[1]][r] - p0) + (double)p[1] * (m->v[t[2]][r] - p0)) +
                       (double)p[2] * (m->v[t[3]][r] - p0));
  }
}

/* ------------------------------------------------------------ quadrature */
typedef struct {
  int degree, n;
  double p[64][3];
  double w[64];
} Rule;

/* symmetric eigen decomposition by cyclic Jacobi (n <= 8), ascending */
static void sym_eig(int n, double a[8][8], double vals[8], double vecs[8][8]) {
  double v[8][8];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) v[i][j] = i == j;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) off += a[p][q] * a[p][q];
    if (off < 1e-300) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        if (fabs(a[p][q]) < 1e-300) continue;
        const double th = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
        const double t = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {
          const double akp = a[k][p], akq = a[k][q];
          a[k][p] = c * akp - s * akq;
          a[k][q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = a[p][k], aqk = a[q][k];
          a[p][k] = c * apk - s * aqk;
          a[q][k] = s * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          const double vkp = v[k][p], vkq = v[k][q];
          v[k][p] = c * vkp - s * vkq;
          v[k][q] = s * vkp + c * vkq;
        }
      }
  }
  int order[8];
  for (int i = 0; i < n; ++i) order[i] = i;
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j)
      if (a[order[j]][order[j]] < a[order[i]][order[i]]) { int s = order[i]; order[i] = order[j]; order[j] = s; }
  for (int j = 0; j < n; ++j) {
    vals[j] = a[order[j]][order[j]];
    for (int k = 0; k < n; ++k) vecs[k][j] = v[k][order[j]];
  }
}

/* Gauss-Jacobi on [0,1], weight (1-x)^alpha (quadrature.cpp:19-57) */
static void gauss_jacobi01(int n, int alpha, double* x, double* w) {
  const double a = alpha, b = 0.0;
  double jac[8][8] = {{0}};
  for (int i = 0; i < n; ++i) {
    double diag;
    if (i == 0) {
      diag = (b - a) / (a + b + 2.0);
    } else {
      const double k = i;
      diag = (b * b - a * a) / ((2.0 * k + a + b) * (2.0 * k + a + b + 2.0));
    }
    jac[i][i] = diag;
    if (i + 1 < n) {
      const double k = i + 1;
      const double num = 4.0 * k * (k + a) * (k + b) * (k + a + b);
      const double den = (2.0 * k + a + b) * (2.0 * k + a + b) * (2.0 * k + a + b + 1.0) * (2.0 * k + a + b - 1.0);
      jac[i][i + 1] = jac[i + 1][i] = sqrt(num / den);
    }
  }
  double vals[8], vecs[8][8];
  sym_eig(n, jac, vals, vecs);
  const double mu0 = pow(2.0, a + 1.0) / (a + 1.0);
  for (int i = 0; i < n; ++i) {
    x[i] = 0.5 * (1.0 + vals[i]);
    w[i] = mu0 * vecs[0][i] * vecs[0][i] / pow(2.0, a + 1.0);
  }
}

static void push_point(Rule* r, double x, double y, double z, double w) {
  r->p[r->n][0] = x; r->p[r->n][1] = y; r->p[r->n][2] = z;
  r->w[r->n] = w;
  ++r->n;
}

static int quadrature(int degree, Rule* r) { /* quadrature.cpp:135-147 */
  memset(r, 0, sizeof(*r));
  r->degree = degree;
  if (degree == 1) {
    push_point(r, 0.25, 0.25, 0.25, 1.0 / 6.0);
  } else if (degree == 2) { /* quadrature.cpp:92-103 */
    const double a = 0.58541019662496845446, b = 0.13819660112501051518, w = 1.0 / 24.0;
    push_point(r, a, b, b, w);
    push_point(r, b, a, b, w);
    push_point(r, b, b, a, w);
    push_point(r, b, b, b, w);
  } else if (degree == 4) { /* Keast, quadrature.cpp:107-131 */
    push_point(r, 0.25, 0.25, 0.25, -148.0 / 11250.0);
    const double a = 11.0 / 14.0, b = 1.0 / 14.0, wa = 343.0 / 45000.0;
    push_point(r, a, b, b, wa);
    push_point(r, b, a, b, wa);
    push_point(r, b, b, a, wa);
    push_point(r, b, b, b, wa);
    const double t = sqrt(5.0 / 14.0), c = 0.25 * (1.0 + t), d = 0.25 * (1.0 - t), wcd = 28.0 / 1125.0;
    const double l[6][4] = {{c, c, d, d}, {c, d, c, d}, {c, d, d, c}, {d, c, c, d}, {d, c, d, c}, {d, d, c, c}};
    for (int i = 0; i < 6; ++i) push_point(r, l[i][1], l[i][2], l[i][3], wcd);
  } else if (degree == 3 || degree == 5 || degree == 6) { /* conical product :66-82 */
    const int n = degree == 3 ? 2 : (degree == 5 ? 3 : 4);
    double x2[8], w2[8], x1[8], w1[8], x0[8], w0[8];
    gauss_jacobi01(n, 2, x2, w2);
    gauss_jacobi01(n, 1, x1, w1);
    gauss_jacobi01(n, 0, x0, w0);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
        for (int k = 0; k < n; ++k) {
          const double x = x2[i], y = x1[j] * (1.0 - x), z = x0[k] * (1.0 - x - y);
          push_point(r, x, y, z, w2[i] * w1[j] * w0[k]);
        }
  } else {
    set_err("quadrature: unsupported degree %d (supported: 1..6)", degree);
    return 1;
  }
  return 0;
}

/* ------------------------------------------------------------ bases */
static const double kGradLambda[4][3] = {{-1, -1, -1}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}};

static void lambda(const double x[3], double l[4]) { /* fespace.cpp:14-16 */
  l[0] = 1.0 - x[0] - x[1] - x[2];
  l[1] = x[0]; l[2] = x[1]; l[3] = x[2];
}

static void basis_nd1(int i, const double x[3], double out[3]) { /* fespace.cpp:102-107 */
  double l[4];
  lambda(x, l);
  const int a = kLocalEdges[i][0], b = kLocalEdges[i][1];
  for (int c = 0; c < 3; ++c) out[c] = l[a] * kGradLambda[b][c] - l[b] * kGradLambda[a][c];
}

static void curl_nd1(int i, double out[3]) { /* fespace.cpp:109-113 */
  const int a = kLocalEdges[i][0], b = kLocalEdges[i][1];
  const double* u = kGradLambda[a];
  const double* v = kGradLambda[b];
  out[0] = 2.0 * (u[1] * v[2] - u[2] * v[1]);
  out[1] = 2.0 * (u[2] * v[0] - u[0] * v[2]);
  out[2] = 2.0 * (u[0] * v[1] - u[1] * v[0]);
}

/* ------------------------------------------------------------ DoF indexer */
typedef struct {
  int32_t owner;
  int16_t x, y, z;
  uint8_t kindClass; /* 0 vertex, 1 + c edge of class c */
  uint8_t flags;     /* bit0 boundary, bit1 canonical dir key-ascending */
} Record;

typedef struct { /* canonical carrier key: sorted (vid, weight) pairs */
  int kind, na, nb;
  int a[4][2], b[4][2];
} Key;

typedef struct {
  Key key;
  i64 value;
  int used;
} Slot;

typedef struct {
  Slot* s;
  size_t cap, count;
} Table;

static uint64_t key_hash(const Key* k) {
  uint64_t h = 1469598103934665603ull ^ (uint64_t)k->kind;
  const int* p = &k->a[0][0];
  for (int i = 0; i < 2 * k->na; ++i) h = (h ^ (uint64_t)(uint32_t)p[i]) * 1099511628211ull;
  h = (h ^ 0xABCDull) * 1099511628211ull;
  p = &k->b[0][0];
  for (int i = 0; i < 2 * k->nb; ++i) h = (h ^ (uint64_t)(uint32_t)p[i]) * 1099511628211ull;
  return h ^ (h >> 29);
}
static int key_eq(const Key* x, const Key* y) {
  return x->kind == y->kind && x->na == y->na && x->nb == y->nb &&
         !memcmp(x->a, y->a, sizeof(int) * 2 * x->na) && !memcmp(x->b, y->b, sizeof(int) * 2 * x->nb);
}
static void table_grow(Table* t);
/* returns existing value, or inserts v and returns -1 */
static i64 table_find_or_insert(Table* t, const Key* k, i64 v) {
  if (2 * (t->count + 1) > t->cap) table_grow(t);
  size_t i = key_hash(k) & (t->cap - 1);
  while (t->s[i].used) {
    if (key_eq(&t->s[i].key, k)) return t->s[i].value;
    i = (i + 1) & (t->cap - 1);
  }
  t->s[i].used = 1;
  t->s[i].key = *k;
  t->s[i].value = v;
  ++t->count;
  return -1;
}
static void table_grow(Table* t) {
  Table n = {calloc(t->cap ? 2 * t->cap : 1024, sizeof(Slot)), t->cap ? 2 * t->cap : 1024, 0};
  for (size_t i = 0; i < t->cap; ++i)
    if (t->s[i].used) table_find_or_insert(&n, &t->s[i].key, t->s[i].value);
  free(t->s);
  *t = n;
}

static int pair_less(const int* x, const int* y) { return x[0] != y[0] ? x[0] < y[0] : x[1] < y[1]; }

/* pack_vertex_key fespace.cpp:124-142 (as a sorted pair list) */
static int vertex_key(const Mesh* m, int macro, int n, const int p[3], int out[4][2]) {
  const int w[4] = {n - p[0] - p[1] - p[2], p[0], p[1], p[2]};
  int k = 0;
  for (int v = 0; v < 4; ++v)
    if (w[v] > 0) { out[k][0] = m->t[macro][v]; out[k][1] = w[v]; ++k; }
  for (int i = 0; i < k; ++i)
    for (int j = i + 1; j < k; ++j)
      if (pair_less(out[j], out[i])) {
        int s0 = out[i][0], s1 = out[i][1];
        out[i][0] = out[j][0]; out[i][1] = out[j][1];
        out[j][0] = s0; out[j][1] = s1;
      }
  return k;
}

/* vertex_key_less fespace.cpp:151-169 */
static int vertex_key_less(const Mesh* m, int macro, int n, const int p[3], const int q[3]) {
  const int* t = m->t[macro];
  int order[4] = {0, 1, 2, 3};
  for (int i = 0; i < 4; ++i)
    for (int j = i + 1; j < 4; ++j)
      if (t[order[j]] < t[order[i]]) { int s = order[i]; order[i] = order[j]; order[j] = s; }
  const int wp[4] = {n - p[0] - p[1] - p[2], p[0], p[1], p[2]};
  const int wq[4] = {n - q[0] - q[1] - q[2], q[0], q[1], q[2]};
  for (int k = 0; k < 4; ++k) {
    const int v = order[k], a = wp[v], b = wq[v];
    if (a > 0 && b > 0) {
      if (a != b) return a < b;
    } else if (a > 0) {
      return 1;
    } else if (b > 0) {
      return 0;
    }
  }
  return 0;
}

static i64 tet_count(i64 k) { return k < 0 ? 0 : (k + 1) * (k + 2) * (k + 3) / 6; }
static i64 lat_index(i64 n, i64 x, i64 y, i64 z) {
  return tet_count(n) - tet_count(n - z) + y * (n - z + 1) - y * (y - 1) / 2 + x;
}

typedef struct {
  int space; /* 0 P1, 2 ND1 */
  const Mesh* mesh;
  int level, n;
  i64 num_dofs;
  Record* rec;          /* sorted by global id */
  uint8_t* interior;
  i64 msize;            /* map entries per macro */
  i64 cstride;          /* ND1 class block */
  i64* map;             /* per macro: +-(id+1), 0 = no carrier */
} Indexer;

static void indexer_free(Indexer* ix) {
  free(ix->rec);
  free(ix->interior);
  free(ix->map);
  memset(ix, 0, sizeof(*ix));
}

static const Record* g_sort_rec;
static int cmp_rec(const void* a, const void* b) {
  const Record* x = g_sort_rec + *(const i64*)a;
  const Record* y = g_sort_rec + *(const i64*)b;
  if (x->owner != y->owner) return x->owner < y->owner ? -1 : 1;
  if (x->z != y->z) return x->z < y->z ? -1 : 1;
  if (x->y != y->y) return x->y < y->y ? -1 : 1;
  if (x->x != y->x) return x->x < y->x ? -1 : 1;
  if (x->kindClass != y->kindClass) return x->kindClass < y->kindClass ? -1 : 1;
  return 0;
}

/* DoFIndexer::DoFIndexer + build + fill_map (fespace.cpp:173-376) */
static int indexer_build(Indexer* ix, int space, const Mesh* mesh, int level) {
  memset(ix, 0, sizeof(*ix));
  ix->space = space;
  ix->mesh = mesh;
  ix->level = level;
  const int n = ix->n = 1 << level;
  if (space == 2 && level < 1) { set_err("ND1 requires level >= 1"); return 1; }
  ix->cstride = tet_count(n - 1);
  ix->msize = space == 0 ? tet_count(n) : 7 * ix->cstride;
  ix->map = calloc((size_t)(ix->msize * mesh->nt), sizeof(i64));
  int* fc = face_counts(mesh);
  size_t cap = 1024, count = 0;
  Record* rec = malloc(sizeof(Record) * cap);
  Table tab = {0};
  for (int m = 0; m < mesh->nt; ++m) {
    i64* map = ix->map + (size_t)m * ix->msize;
    const int* bf = fc + 4 * m; /* boundary face opposite local vertex v: count == 1 */
    if (space == 0) {
      for (int z = 0; z <= n; ++z)
        for (int y = 0; y <= n - z; ++y)
          for (int x = 0; x <= n - z - y; ++x) {
            const int p[3] = {x, y, z};
            const int w[4] = {n - x - y - z, x, y, z};
            const int iface = w[0] == 0 || w[1] == 0 || w[2] == 0 || w[3] == 0;
            uint8_t flags = 0;
            for (int v = 0; v < 4; ++v)
              if (bf[v] == 1 && w[v] == 0) flags |= 1;
            i64 ci = (i64)count;
            int create = 1;
            if (iface) {
              Key k = {0};
              k.kind = 0;
              k.na = vertex_key(mesh, m, n, p, k.a);
              const i64 prev = table_find_or_insert(&tab, &k, ci);
              if (prev >= 0) { ci = prev; create = 0; rec[prev].flags |= flags & 1; }
            }
            if (create) {
              if (count == cap) rec = realloc(rec, sizeof(Record) * (cap *= 2));
              rec[count++] = (Record){m, (int16_t)x, (int16_t)y, (int16_t)z, 0, flags};
            }
            map[lat_index(n, x, y, z)] = ci + 1;
          }
    } else {
      for (int c = 0; c < 7; ++c)
        for (int z = 0; z <= n; ++z)
          for (int y = 0; y <= n - z; ++y)
            for (int x = 0; x <= n - z - y; ++x) {
              const int p[3] = {x, y, z};
              const int q[3] = {x + kEdgeDirs[c][0], y + kEdgeDirs[c][1], z + kEdgeDirs[c][2]};
              if (q[0] < 0 || q[1] < 0 || q[2] < 0 || q[0] + q[1] + q[2] > n) continue;
              const int wp[4] = {n - p[0] - p[1] - p[2], p[0], p[1], p[2]};
              const int wq[4] = {n - q[0] - q[1] - q[2], q[0], q[1], q[2]};
              int iface = 0;
              for (int v = 0; v < 4 && !iface; ++v) iface = wp[v] == 0 && wq[v] == 0;
              uint8_t flags = 0;
              for (int v = 0; v < 4; ++v)
                if (bf[v] == 1 && wp[v] == 0 && wq[v] == 0) flags |= 1;
              const int asc = vertex_key_less(mesh, m, n, p, q);
              if (asc) flags |= 2;
              i64 ci = (i64)count;
              int create = 1;
              if (iface) {
                Key k = {0};
                int ka[4][2], kb[4][2];
                const int na = vertex_key(mesh, m, n, p, ka), nb = vertex_key(mesh, m, n, q, kb);
                /* canonical order of the two endpoint keys */
                int less = 0, i = 0;
                while (i < na && i < nb && !memcmp(ka[i], kb[i], sizeof(ka[i]))) ++i;
                if (i < na && i < nb) less = pair_less(ka[i], kb[i]);
                else less = na < nb;
                k.kind = 1;
                if (less) { k.na = na; k.nb = nb; memcpy(k.a, ka, sizeof ka); memcpy(k.b, kb, sizeof kb); }
                else { k.na = nb; k.nb = na; memcpy(k.a, kb, sizeof kb); memcpy(k.b, ka, sizeof ka); }
                const i64 prev = table_find_or_insert(&tab, &k, ci);
                if (prev >= 0) { ci = prev; create = 0; rec[prev].flags |= flags & 1; }
              }
              if (create) {
                if (count == cap) rec = realloc(rec, sizeof(Record) * (cap *= 2));
                rec[count++] = (Record){m, (int16_t)x, (int16_t)y, (int16_t)z, (uint8_t)(1 + c), flags};
              }
              /* slot by anchor = componentwise min of p, q (this port's map layout) */
              const int ax = p[0] < q[0] ? p[0] : q[0], ay = p[1] < q[1] ? p[1] : q[1],
                        az = p[2] < q[2] ? p[2] : q[2];
              map[c * ix->cstride + lat_index(n - 1, ax, ay, az)] = asc ? ci + 1 : -(ci + 1);
            }
    }
  }
  free(tab.s);
  free(fc);
  /* global numbering: sort by (owner, z, y, x, kindClass) (fespace.cpp:283-297) */
  i64* order = malloc(sizeof(i64) * (count ? count : 1));
  for (size_t i = 0; i < count; ++i) order[i] = (i64)i;
  g_sort_rec = rec;
  qsort(order, count, sizeof(i64), cmp_rec);
  i64* rank = malloc(sizeof(i64) * (count ? count : 1));
  for (size_t id = 0; id < count; ++id) rank[order[id]] = (i64)id;
  ix->rec = malloc(sizeof(Record) * (count ? count : 1));
  for (size_t id = 0; id < count; ++id) ix->rec[id] = rec[order[id]];
  ix->num_dofs = (i64)count;
  ix->interior = malloc(count ? count : 1);
  for (size_t id = 0; id < count; ++id) ix->interior[id] = (ix->rec[id].flags & 1) ? 0 : 1;
  for (i64 i = 0; i < ix->msize * mesh->nt; ++i) {
    const i64 v = ix->map[i];
    if (v > 0) ix->map[i] = rank[v - 1] + 1;
    else if (v < 0) ix->map[i] = -(rank[-v - 1] + 1);
  }
  free(order);
  free(rank);
  free(rec);
  return 0;
}

/* local_dofs fespace.cpp:393-430 */
static int local_dofs(const Indexer* ix, int macro, int o, int x, int y, int z, i64* ids, double* signs) {
  const int n = ix->n;
  const i64* map = ix->map + (size_t)macro * ix->msize;
  int v[4][3];
  for (int i = 0; i < 4; ++i)
    for (int c = 0; c < 3; ++c) v[i][c] = (c == 0 ? x : c == 1 ? y : z) + kOffsets[o][i][c];
  if (ix->space == 0) {
    for (int i = 0; i < 4; ++i) {
      const i64 e = map[lat_index(n, v[i][0], v[i][1], v[i][2])];
      ids[i] = (e < 0 ? -e : e) - 1;
      signs[i] = 1.0;
    }
    return 4;
  }
  for (int le = 0; le < 6; ++le) {
    const int* pa = v[kLocalEdges[le][0]];
    const int* pb = v[kLocalEdges[le][1]];
    const int d[3] = {pb[0] - pa[0], pb[1] - pa[1], pb[2] - pa[2]};
    int flipped;
    const int c = edge_class(d, &flipped);
    const int ax = pa[0] < pb[0] ? pa[0] : pb[0], ay = pa[1] < pb[1] ? pa[1] : pb[1],
              az = pa[2] < pb[2] ? pa[2] : pb[2];
    const i64 e = map[c * ix->cstride + lat_index(n - 1, ax, ay, az)];
    ids[le] = (e < 0 ? -e : e) - 1;
    double s = e > 0 ? 1.0 : -1.0;
    if (flipped) s = -s;
    signs[le] = s;
  }
  return 6;
}

/* ------------------------------------------------------------ forms */
typedef struct {
  Mesh mesh;
  int form; /* 0 P1, 1 P1K (harness), 2 N1 */
  int level;
  Indexer primary;
  Indexer coeff; /* P1 indexer of the coefficients (N1); P1/P1K use primary */
} Port;

/* StarTables forms.cpp:69-131 for one (macro, orientation, rule) */
static void stars(const Port* P, int macro, int o, const Rule* rule, double* starA, double* starB) {
  double J[3][3], det, jinvT[3][3];
  micro_jacobian(&P->mesh, macro, P->level, o, J, &det);
  const double absdet = fabs(det);
  inverse_transpose(J, jinvT);
  const int nloc = P->form == 2 ? 6 : 4;
  for (int q = 0; q < rule->n; ++q) {
    const double wdet = rule->w[q] * absdet;
    if (P->form == 2) {
      double curls[6][3], vals[6][3];
      for (int i = 0; i < 6; ++i) {
        double cr[3], b[3];
        curl_nd1(i, cr);
        for (int r = 0; r < 3; ++r)
          curls[i][r] = (1.0 / det) * (J[r][0] * cr[0] + J[r][1] * cr[1] + J[r][2] * cr[2]);
        basis_nd1(i, rule->p[q], b);
        for (int r = 0; r < 3; ++r) vals[i][r] = jinvT[r][0] * b[0] + jinvT[r][1] * b[1] + jinvT[r][2] * b[2];
      }
      for (int j = 0; j < nloc; ++j)
        for (int i = 0; i < nloc; ++i) {
          starA[(q * nloc + j) * nloc + i] =
              wdet * (curls[i][0] * curls[j][0] + curls[i][1] * curls[j][1] + curls[i][2] * curls[j][2]);
          starB[(q * nloc + j) * nloc + i] =
              wdet * (vals[i][0] * vals[j][0] + vals[i][1] * vals[j][1] + vals[i][2] * vals[j][2]);
        }
    } else {
      double g[4][3];
      for (int i = 0; i < 4; ++i)
        for (int r = 0; r < 3; ++r)
          g[i][r] = jinvT[r][0] * kGradLambda[i][0] + jinvT[r][1] * kGradLambda[i][1] + jinvT[r][2] * kGradLambda[i][2];
      for (int j = 0; j < nloc; ++j)
        for (int i = 0; i < nloc; ++i)
          starA[(q * nloc + j) * nloc + i] = wdet * (g[i][0] * g[j][0] + g[i][1] * g[j][1] + g[i][2] * g[j][2]);
    }
  }
}

static double alpha_fn(const double p[3]) { return 1.0 + p[0] * p[0] + p[1] * p[1]; }
static double beta_fn(const double p[3]) { return 2.0 + sin(M_PI * p[2]); }
static double k_fn(const double p[3]) {
  return 1.0 + 0.5 * sin(2.0 * M_PI * p[0]) * cos(2.0 * M_PI * p[1]) * (1.0 + p[2]);
}

static void dof_geometry(const Indexer* ix, i64 id, int* kind, double a[3], double b[3]) { /* fespace.cpp:432-451 */
  const Record* r = &ix->rec[id];
  const int base[3] = {r->x, r->y, r->z};
  if (r->kindClass == 0) {
    *kind = 0;
    lattice_to_world(ix->mesh, r->owner, ix->level, base, a);
    memcpy(b, a, sizeof(double) * 3);
    return;
  }
  *kind = 1;
  const int c = r->kindClass - 1;
  const int tip[3] = {base[0] + kEdgeDirs[c][0], base[1] + kEdgeDirs[c][1], base[2] + kEdgeDirs[c][2]};
  double pa[3], pb[3];
  lattice_to_world(ix->mesh, r->owner, ix->level, base, pa);
  lattice_to_world(ix->mesh, r->owner, ix->level, tip, pb);
  if (!(r->flags & 2)) { memcpy(a, pb, sizeof pa); memcpy(b, pa, sizeof pa); }
  else { memcpy(a, pa, sizeof pa); memcpy(b, pb, sizeof pb); }
}

/* ------------------------------------------------------------ C API */
void* port_create(const char* mesh, const char* form, int level) {
  Port* P = calloc(1, sizeof(Port));
  if (mesh_by_name(&P->mesh, mesh)) { free(P); return NULL; }
  if (!strcmp(form, "P1")) P->form = 0;
  else if (!strcmp(form, "P1K")) P->form = 1;
  else if (!strcmp(form, "N1")) P->form = 2;
  else { set_err("unknown form '%s' (expected P1, P1K or N1)", form); mesh_free(&P->mesh); free(P); return NULL; }
  if (level < 0) { set_err("DoFIndexer: negative level"); mesh_free(&P->mesh); free(P); return NULL; }
  P->level = level;
  if (indexer_build(&P->primary, P->form == 2 ? 2 : 0, &P->mesh, level)) { mesh_free(&P->mesh); free(P); return NULL; }
  if (P->form == 2 && indexer_build(&P->coeff, 0, &P->mesh, level)) {
    indexer_free(&P->primary); mesh_free(&P->mesh); free(P); return NULL;
  }
  return P;
}

void port_destroy(void* h) {
  Port* P = h;
  if (!P) return;
  indexer_free(&P->primary);
  indexer_free(&P->coeff);
  mesh_free(&P->mesh);
  free(P);
}

long long port_num_dofs(void* h) { return ((Port*)h)->primary.num_dofs; }
int port_num_macros(void* h) { return ((Port*)h)->mesh.nt; }

int port_dof_geometry(void* h, unsigned char* kind, double* a, double* b) {
  const Indexer* ix = &((Port*)h)->primary;
  for (i64 id = 0; id < ix->num_dofs; ++id) {
    int k;
    dof_geometry(ix, id, &k, a + 3 * id, b + 3 * id);
    kind[id] = (unsigned char)k;
  }
  return 0;
}

int port_interior(void* h, unsigned char* out) {
  const Indexer* ix = &((Port*)h)->primary;
  memcpy(out, ix->interior, (size_t)ix->num_dofs);
  return 0;
}

static const Indexer* coeff_ix(const Port* P) { return P->form == 2 ? &P->coeff : &P->primary; }

long long port_coeff_num_dofs(void* h) { return coeff_ix(h)->num_dofs; }

int port_coeff_geometry(void* h, double* a) {
  const Indexer* ix = coeff_ix(h);
  for (i64 id = 0; id < ix->num_dofs; ++id) {
    int k;
    double b[3];
    dof_geometry(ix, id, &k, a + 3 * id, b);
  }
  return 0;
}

int port_interpolate(void* h, int which, double* out) { /* interpolate fespace.cpp:494-506 */
  const Indexer* ix = coeff_ix(h);
  for (i64 id = 0; id < ix->num_dofs; ++id) {
    int k;
    double a[3], b[3];
    dof_geometry(ix, id, &k, a, b);
    out[id] = which == 0 ? alpha_fn(a) : which == 1 ? beta_fn(a) : k_fn(a);
  }
  return 0;
}

/* FormSystem::apply forms.cpp:195-255 (Replace semantics, sawtooth order),
 * restricted to macros with mask[m] != 0 (all when mask == NULL). */
static int apply_impl(Port* P, const double* v, const double* c0, const double* c1, int degree,
                      const unsigned char* mask, double* w) {
  Rule rule;
  /* reference_apply: min(exactDegree + 2, 6): P1 -> 2, N1 -> 5 (forms.cpp:257-260) */
  if (quadrature(degree > 0 ? degree : (P->form == 2 ? 5 : 2), &rule)) return 1;
  if (P->form != 0 && !c0) { set_err("form expects coefficient field(s)"); return 1; }
  if (P->form == 2 && !c1) { set_err("form N1 expects 2 coefficient fields"); return 1; }
  const int nloc = P->form == 2 ? 6 : 4, nq = rule.n, n = P->primary.n;
  memset(w, 0, sizeof(double) * (size_t)P->primary.num_dofs);
  double* starA = malloc(sizeof(double) * (size_t)nq * nloc * nloc);
  double* starB = malloc(sizeof(double) * (size_t)nq * nloc * nloc);
  double phi[64][4];
  for (int q = 0; q < nq; ++q) lambda(rule.p[q], phi[q]); /* coeffBasis[q][m] (forms.cpp:119-127) */
  const Indexer* kix = coeff_ix(P);
  for (int m = 0; m < P->mesh.nt; ++m) {
    if (mask && !mask[m]) continue;
    for (int o = 0; o < 6; ++o) {
      stars(P, m, o, &rule, starA, starB);
      const int B = loop_bound(o, n);
      for (int z = 0; z < B; ++z)
        for (int y = 0; y < loop_bound(o, n - z); ++y)
          for (int x = 0; x < loop_bound(o, n - z - y); ++x) {
            i64 ids[6], kids[6];
            double sg[6], ksg[6], aq[64], bq[64], entries[36];
            local_dofs(&P->primary, m, o, x, y, z, ids, sg);
            if (P->form != 0) {
              local_dofs(kix, m, o, x, y, z, kids, ksg);
              for (int q = 0; q < nq; ++q) {
                double a = 0.0, b = 0.0;
                for (int km = 0; km < 4; ++km) {
                  a += c0[kids[km]] * phi[q][km];
                  if (P->form == 2) b += c1[kids[km]] * phi[q][km];
                }
                aq[q] = a;
                bq[q] = b;
              }
            } else {
              for (int q = 0; q < nq; ++q) aq[q] = 1.0;
            }
            if (P->form == 1) {
              /* config-2 harness: A_e = local_matrix(e, {}, rule) (cq = 1),
               * kbar = 6 * sum_q w_q k_q */
              for (int k = 0; k < 16; ++k) entries[k] = 0.0;
              for (int q = 0; q < nq; ++q)
                for (int k = 0; k < 16; ++k) entries[k] += 1.0 * starA[q * 16 + k];
              double kbar = 0.0;
              for (int q = 0; q < nq; ++q) kbar += rule.w[q] * aq[q];
              kbar *= 6.0;
              for (int j = 0; j < 4; ++j) {
                double acc = 0.0;
                for (int i = 0; i < 4; ++i) acc += kbar * entries[j * 4 + i] * v[ids[i]];
                w[ids[j]] += acc;
              }
              continue;
            }
            for (int k = 0; k < nloc * nloc; ++k) entries[k] = 0.0;
            for (int q = 0; q < nq; ++q) {
              const double* sa = starA + (size_t)q * nloc * nloc;
              for (int k = 0; k < nloc * nloc; ++k) entries[k] += aq[q] * sa[k];
              if (P->form == 2) {
                const double* sb = starB + (size_t)q * nloc * nloc;
                for (int k = 0; k < nloc * nloc; ++k) entries[k] += bq[q] * sb[k];
              }
            }
            for (int j = 0; j < nloc; ++j) {
              double acc = 0.0;
              for (int i = 0; i < nloc; ++i) acc += entries[j * nloc + i] * sg[i] * v[ids[i]];
              w[ids[j]] += sg[j] * acc;
            }
          }
    }
  }
  free(starA);
  free(starB);
  return 0;
}

int port_apply(void* h, const double* v, const double* c0, const double* c1, int degree, double* w,
               double* seconds) {
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  const int rc = apply_impl(h, v, c0, c1, degree, NULL, w);
  clock_gettime(CLOCK_MONOTONIC, &t1);
  if (seconds) *seconds = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
  return rc;
}

int port_apply_macros(void* h, const double* v, const double* c0, const double* c1, int degree,
                      const unsigned char* macro_mask, double* w) {
  return apply_impl(h, v, c0, c1, degree, macro_mask, w);
}
