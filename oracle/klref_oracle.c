/*
 * TEST INFRASTRUCTURE — CPU restatement of the reference hot path (oracle).
 * Not product code: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it, as the checker.
 *
 * Plain C restatement of the 2-d path of arXiv 2508.06049's reference
 * (/root/reference/proj), written as sequential loops in the reference's own
 * order so it reproduces the patched reference bit for bit:
 *   hierarchy groups / ownership          proj/src/hhg.cpp:48-144
 *   boundary_group (D2 fixed)             proj/src/hhg.cpp:163-174
 *   interface_sync, dot_unique            proj/src/hhg.cpp:206-257
 *   element matrices (D1 fixed), stencil  proj/src/fem.cpp:30-46, 62-93
 *   apply (element scatter)               proj/src/fem.cpp:95-126
 *   partial_row                           proj/src/fem.cpp:128-173
 *   assemble_rhs, Dirichlet values        proj/src/fem.cpp:175-241
 *   l2_norm, local_l2_norms               proj/src/fem.cpp:320-356
 *   prolongate, restrict_transpose        proj/src/multigrid.cpp:22-111
 *   gauss_seidel, residual, cg_level0     proj/src/multigrid.cpp:127-229
 *   v_cycle, fmg (FinestPolicy::None)     proj/src/multigrid.cpp:231-279
 *   error_estimate                        proj/src/estimator.cpp:8-45
 * Pinned against the reference itself: tests/test_oracle_cpu.py checks every
 * output against the sha256 / values of tests/golden (oracle/_ref runs).
 * Compile without -march / -ffast-math (no FMA contraction).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MAXL 12

typedef struct {
  int group_start;
  int owner;
  int domain_boundary;
} o_edge;

typedef struct {
  int corner_group[3];
  int corner_owner[3];
  int corner_boundary[3];
  o_edge edge[3];
} o_macro_level;

typedef struct {
  int n, S;
  int ngroups;
  int* gptr;   /* ngroups + 1 */
  int* mslot;  /* members */
  int* midx;
  int* mi;
  int* mj;
  o_macro_level* macros;
  long long dofs;
  double* ku; /* 9 per macro (stiffness up) */
  double* kd; /* stiffness down */
  double* mu; /* mass up */
  double* md; /* mass down */
  double* st; /* 7 per macro */
} o_level;

typedef struct {
  int M, L, nv;
  double* vx;
  double* vy;
  int* vbnd;
  int* tri; /* 3 per macro, oriented */
  double* area;
  o_level lev[MAXL + 1];
} oh2d;

static const int kEdges[3][2] = {{0, 1}, {0, 2}, {1, 2}};

static int lat(int n, int i, int j) { return j * (n + 1) - (j * (j - 1)) / 2 + i; }
static int latsize(int n) { return (n + 1) * (n + 2) / 2; }

static double signed_area(const oh2d* h, int a, int b, int c) {
  return 0.5 * ((h->vx[b] - h->vx[a]) * (h->vy[c] - h->vy[a]) - (h->vy[b] - h->vy[a]) * (h->vx[c] - h->vx[a]));
}

/* stiffness_matrix with the D1 fix (|area|), proj/src/fem.cpp:30-41 */
static void stiffness_matrix(double p0x, double p0y, double p1x, double p1y, double p2x, double p2y, double* k) {
  const double area2 = (p1x - p0x) * (p2y - p0y) - (p1y - p0y) * (p2x - p0x);
  const double area = 0.5 * fabs(area2);
  const double gx[3] = {-(p2y - p1y) / area2, -(p0y - p2y) / area2, -(p1y - p0y) / area2};
  const double gy[3] = {(p2x - p1x) / area2, (p0x - p2x) / area2, (p1x - p0x) / area2};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) k[3 * i + j] = area * (gx[i] * gx[j] + gy[i] * gy[j]);
}

static void mass_matrix(double area, double* k) {
  const double d = area / 6.0, o = area / 12.0;
  k[0] = d; k[1] = o; k[2] = o;
  k[3] = o; k[4] = d; k[5] = o;
  k[6] = o; k[7] = o; k[8] = d;
}

/* node_coordinates, proj/src/hhg.cpp:146-154 */
static void node_xy(const oh2d* h, int slot, int l, int i, int j, double* x, double* y) {
  const int n = h->lev[l].n;
  const int* v = h->tri + 3 * slot;
  const double xi = (double)i / n, yj = (double)j / n;
  *x = h->vx[v[0]] + xi * (h->vx[v[1]] - h->vx[v[0]]) + yj * (h->vx[v[2]] - h->vx[v[0]]);
  *y = h->vy[v[0]] + xi * (h->vy[v[1]] - h->vy[v[0]]) + yj * (h->vy[v[2]] - h->vy[v[0]]);
}

/* boundary_group with the D2 fix, proj/src/hhg.cpp:163-174 */
static int boundary_group(const oh2d* h, int slot, int l, int i, int j) {
  const o_level* lv = &h->lev[l];
  const int n = lv->n;
  const o_macro_level* ml = &lv->macros[slot];
  const int* ids = h->tri + 3 * slot;
  if (i == 0 && j == 0) return ml->corner_group[0];
  if (i == n && j == 0) return ml->corner_group[1];
  if (i == 0 && j == n) return ml->corner_group[2];
  if (j == 0) return ml->edge[0].group_start + ((ids[0] < ids[1] ? i : n - i) - 1);
  if (i == 0) return ml->edge[1].group_start + ((ids[0] < ids[2] ? j : n - j) - 1);
  if (i + j == n) return ml->edge[2].group_start + ((ids[1] < ids[2] ? j : n - j) - 1);
  return -1;
}

static int on_domain_boundary(const oh2d* h, int slot, int l, int i, int j) {
  const o_level* lv = &h->lev[l];
  const int n = lv->n;
  const o_macro_level* ml = &lv->macros[slot];
  if (i == 0 && j == 0) return ml->corner_boundary[0];
  if (i == n && j == 0) return ml->corner_boundary[1];
  if (i == 0 && j == n) return ml->corner_boundary[2];
  if (j == 0) return ml->edge[0].domain_boundary;
  if (i == 0) return ml->edge[1].domain_boundary;
  if (i + j == n) return ml->edge[2].domain_boundary;
  return 0;
}

static int owns_boundary_node(const oh2d* h, int slot, int l, int i, int j) {
  const o_level* lv = &h->lev[l];
  const int n = lv->n;
  const o_macro_level* ml = &lv->macros[slot];
  if (i == 0 && j == 0) return ml->corner_owner[0];
  if (i == n && j == 0) return ml->corner_owner[1];
  if (i == 0 && j == n) return ml->corner_owner[2];
  if (j == 0) return ml->edge[0].owner;
  if (i == 0) return ml->edge[1].owner;
  if (i + j == n) return ml->edge[2].owner;
  return 1;
}

void o2_free(oh2d* h) {
  if (!h) return;
  for (int l = 0; l <= h->L; ++l) {
    o_level* lv = &h->lev[l];
    free(lv->gptr); free(lv->mslot); free(lv->midx); free(lv->mi); free(lv->mj); free(lv->macros);
    free(lv->ku); free(lv->kd); free(lv->mu); free(lv->md); free(lv->st);
  }
  free(h->vx); free(h->vy); free(h->vbnd); free(h->tri); free(h->area);
  free(h);
}

/* vertex / edge incidence lists sorted like the reference's std::map keys */
typedef struct { int key0, key1, slot, c; } o_use;

static int cmp_use(const void* a, const void* b) {
  const o_use* x = (const o_use*)a;
  const o_use* y = (const o_use*)b;
  if (x->key0 != y->key0) return x->key0 < y->key0 ? -1 : 1;
  if (x->key1 != y->key1) return x->key1 < y->key1 ? -1 : 1;
  if (x->slot != y->slot) return x->slot < y->slot ? -1 : 1;
  return x->c < y->c ? -1 : (x->c > y->c);
}

/* GridHierarchy::build, proj/src/hhg.cpp:48-144, plus OperatorP1 matrices */
oh2d* o2_build(int nv, const double* xy, int ne, const int* tri, int L) {
  if (nv <= 0 || ne <= 0 || L < 0 || L > MAXL) return NULL;
  oh2d* h = (oh2d*)calloc(1, sizeof(oh2d));
  h->M = ne;
  h->L = L;
  h->nv = nv;
  h->vx = (double*)malloc(sizeof(double) * nv);
  h->vy = (double*)malloc(sizeof(double) * nv);
  h->vbnd = (int*)calloc(nv, sizeof(int));
  h->tri = (int*)malloc(sizeof(int) * 3 * ne);
  h->area = (double*)malloc(sizeof(double) * ne);
  for (int v = 0; v < nv; ++v) {
    h->vx[v] = xy[2 * v];
    h->vy[v] = xy[2 * v + 1];
  }
  for (int e = 0; e < ne; ++e) {
    int a = tri[3 * e], b = tri[3 * e + 1], c = tri[3 * e + 2];
    if (signed_area(h, a, b, c) < 0.0) { int t = b; b = c; c = t; } /* orient_positive */
    h->tri[3 * e] = a; h->tri[3 * e + 1] = b; h->tri[3 * e + 2] = c;
    h->area[e] = signed_area(h, a, b, c);
  }
  /* uses */
  o_use* vuse = (o_use*)malloc(sizeof(o_use) * 3 * ne);
  o_use* euse = (o_use*)malloc(sizeof(o_use) * 3 * ne);
  for (int s = 0; s < ne; ++s)
    for (int c = 0; c < 3; ++c) {
      o_use u = {h->tri[3 * s + c], 0, s, c};
      vuse[3 * s + c] = u;
      const int a = h->tri[3 * s + kEdges[c][0]], b = h->tri[3 * s + kEdges[c][1]];
      o_use w = {a < b ? a : b, a < b ? b : a, s, c};
      euse[3 * s + c] = w;
    }
  qsort(vuse, 3 * ne, sizeof(o_use), cmp_use);
  qsort(euse, 3 * ne, sizeof(o_use), cmp_use);
  /* vertex boundary flags from edges with one use (rebuild_facets, macro_mesh.cpp:306-318) */
  int nvg = 0, neg = 0;
  for (int k = 0; k < 3 * ne;) {
    int k2 = k;
    while (k2 < 3 * ne && euse[k2].key0 == euse[k].key0 && euse[k2].key1 == euse[k].key1) ++k2;
    if (k2 - k == 1) h->vbnd[euse[k].key0] = h->vbnd[euse[k].key1] = 1;
    ++neg;
    k = k2;
  }
  for (int k = 0; k < 3 * ne;) {
    int k2 = k;
    while (k2 < 3 * ne && vuse[k2].key0 == vuse[k].key0) ++k2;
    ++nvg;
    k = k2;
  }
  for (int l = 0; l <= L; ++l) {
    o_level* lv = &h->lev[l];
    const int n = 1 << l;
    lv->n = n;
    lv->S = latsize(n);
    lv->macros = (o_macro_level*)calloc(ne, sizeof(o_macro_level));
    lv->ngroups = nvg + neg * (n - 1);
    lv->gptr = (int*)malloc(sizeof(int) * (lv->ngroups + 1));
    const int maxm = 3 * ne * (n + 1);
    lv->mslot = (int*)malloc(sizeof(int) * maxm);
    lv->midx = (int*)malloc(sizeof(int) * maxm);
    lv->mi = (int*)malloc(sizeof(int) * maxm);
    lv->mj = (int*)malloc(sizeof(int) * maxm);
    int g = 0, m = 0;
    lv->gptr[0] = 0;
    const int cidx[3] = {lat(n, 0, 0), lat(n, n, 0), lat(n, 0, n)};
    const int cij[3][2] = {{0, 0}, {n, 0}, {0, n}};
    for (int k = 0; k < 3 * ne;) { /* vertex groups, proj/src/hhg.cpp:95-109 */
      int k2 = k;
      while (k2 < 3 * ne && vuse[k2].key0 == vuse[k].key0) ++k2;
      for (int q = k; q < k2; ++q) {
        const int s = vuse[q].slot, c = vuse[q].c;
        lv->mslot[m] = s; lv->midx[m] = cidx[c]; lv->mi[m] = cij[c][0]; lv->mj[m] = cij[c][1]; ++m;
        lv->macros[s].corner_group[c] = g;
        lv->macros[s].corner_boundary[c] = h->vbnd[vuse[q].key0];
      }
      lv->macros[vuse[k].slot].corner_owner[vuse[k].c] = 1;
      lv->gptr[++g] = m;
      k = k2;
    }
    for (int k = 0; k < 3 * ne;) { /* edge groups, proj/src/hhg.cpp:111-132 */
      int k2 = k;
      while (k2 < 3 * ne && euse[k2].key0 == euse[k].key0 && euse[k2].key1 == euse[k].key1) ++k2;
      const int bnd = (k2 - k) == 1;
      const int start = g;
      for (int s = 1; s <= n - 1; ++s) {
        for (int q = k; q < k2; ++q) {
          const int slot = euse[q].slot, le = euse[q].c;
          const int first = h->tri[3 * slot + kEdges[le][0]];
          const int t = (first == euse[q].key0) ? s : n - s;
          const int ii = le == 0 ? t : (le == 1 ? 0 : n - t);
          const int jj = le == 0 ? 0 : t;
          lv->mslot[m] = slot; lv->midx[m] = lat(n, ii, jj); lv->mi[m] = ii; lv->mj[m] = jj; ++m;
        }
        lv->gptr[++g] = m;
      }
      for (int q = k; q < k2; ++q) {
        o_edge* info = &lv->macros[euse[q].slot].edge[euse[q].c];
        info->group_start = start;
        info->owner = (q == k);
        info->domain_boundary = bnd;
      }
      k = k2;
    }
    lv->dofs = (long long)nvg + (long long)neg * (n - 1) + (long long)ne * ((long long)(n - 1) * (n - 2) / 2);
    /* OperatorP1 ctor, proj/src/fem.cpp:62-93 */
    lv->ku = (double*)calloc(9 * ne, sizeof(double));
    lv->kd = (double*)calloc(9 * ne, sizeof(double));
    lv->mu = (double*)calloc(9 * ne, sizeof(double));
    lv->md = (double*)calloc(9 * ne, sizeof(double));
    lv->st = (double*)calloc(7 * ne, sizeof(double));
  }
  free(vuse);
  free(euse);
  for (int l = 0; l <= L; ++l) {
    o_level* lv = &h->lev[l];
    const int n = lv->n;
    for (int s = 0; s < ne; ++s) {
      double p[4][2];
      node_xy(h, s, l, 0, 0, &p[0][0], &p[0][1]);
      node_xy(h, s, l, 1, 0, &p[1][0], &p[1][1]);
      node_xy(h, s, l, 0, 1, &p[2][0], &p[2][1]);
      double* ku = lv->ku + 9 * s;
      double* kd = lv->kd + 9 * s;
      stiffness_matrix(p[0][0], p[0][1], p[1][0], p[1][1], p[2][0], p[2][1], ku);
      if (n >= 2) {
        node_xy(h, s, l, 1, 1, &p[3][0], &p[3][1]);
        stiffness_matrix(p[1][0], p[1][1], p[2][0], p[2][1], p[3][0], p[3][1], kd);
      }
      const double cell_area = h->area[s] / ((double)n * n);
      mass_matrix(cell_area, lv->mu + 9 * s);
      if (n >= 2) mass_matrix(cell_area, lv->md + 9 * s);
      double* st = lv->st + 7 * s;
      st[0] = ku[0] + ku[4] + ku[8] + kd[0] + kd[4] + kd[8];
      st[1] = ku[1] + kd[5];
      st[2] = ku[3] + kd[7];
      st[3] = ku[2] + kd[2];
      st[4] = ku[6] + kd[6];
      st[5] = ku[5] + kd[1];
      st[6] = ku[7] + kd[3];
    }
  }
  return h;
}

int o2_num_macros(const oh2d* h) { return h->M; }
int o2_level_size(const oh2d* h, int l) { return h->M * h->lev[l].S; }
long long o2_dofs(const oh2d* h, int l) { return h->lev[l].dofs; }

/* interface_sync, proj/src/hhg.cpp:206-225 */
void o2_interface_sync(const oh2d* h, int l, double* f, int additive) {
  const o_level* lv = &h->lev[l];
  const int S = lv->S;
  for (int g = 0; g < lv->ngroups; ++g) {
    const int b = lv->gptr[g], e = lv->gptr[g + 1];
    if (e - b < 2) continue;
    if (!additive) {
      const double v = f[lv->mslot[b] * S + lv->midx[b]];
      for (int k = b + 1; k < e; ++k) f[lv->mslot[k] * S + lv->midx[k]] = v;
    } else {
      double sum = 0.0;
      for (int k = b; k < e; ++k) sum += f[lv->mslot[k] * S + lv->midx[k]];
      for (int k = b; k < e; ++k) f[lv->mslot[k] * S + lv->midx[k]] = sum;
    }
  }
}

static int edge_lattice_index(int n, int le, int t) {
  if (le == 0) return lat(n, t, 0);
  if (le == 1) return lat(n, 0, t);
  return lat(n, n - t, t);
}

/* dot_unique, proj/src/hhg.cpp:227-257 */
double o2_dot_unique(const oh2d* h, int l, const double* a, const double* b) {
  const o_level* lv = &h->lev[l];
  const int n = lv->n, S = lv->S;
  double sum = 0.0;
  for (int s = 0; s < h->M; ++s) {
    const double* xa = a + (size_t)s * S;
    const double* xb = b + (size_t)s * S;
    for (int j = 1; j < n; ++j) {
      const int base = lat(n, 0, j);
      for (int i = 1; i < n - j; ++i) sum += xa[base + i] * xb[base + i];
    }
    const o_macro_level* ml = &lv->macros[s];
    const int ci[3] = {lat(n, 0, 0), lat(n, n, 0), lat(n, 0, n)};
    for (int c = 0; c < 3; ++c)
      if (ml->corner_owner[c]) sum += xa[ci[c]] * xb[ci[c]];
    for (int le = 0; le < 3; ++le) {
      if (!ml->edge[le].owner) continue;
      for (int t = 1; t <= n - 1; ++t) {
        const int idx = edge_lattice_index(n, le, t);
        sum += xa[idx] * xb[idx];
      }
    }
  }
  return sum;
}

/* OperatorP1::apply (element scatter), proj/src/fem.cpp:95-126 */
void o2_apply(const oh2d* h, int l, int mass, const double* x, double* y) {
  const o_level* lv = &h->lev[l];
  const int n = lv->n, S = lv->S;
  for (int s = 0; s < h->M; ++s) {
    const double* xm = x + (size_t)s * S;
    double* ym = y + (size_t)s * S;
    memset(ym, 0, sizeof(double) * S);
    const double* ku = (mass ? lv->mu : lv->ku) + 9 * s;
    const double* kd = (mass ? lv->md : lv->kd) + 9 * s;
    for (int j = 0; j < n; ++j) {
      const int r0 = lat(n, 0, j), r1 = lat(n, 0, j + 1);
      for (int i = 0; i < n - j; ++i) {
        const int a = r0 + i, b = r0 + i + 1, c = r1 + i;
        const double xa = xm[a], xb = xm[b], xc = xm[c];
        ym[a] += ku[0] * xa + ku[1] * xb + ku[2] * xc;
        ym[b] += ku[3] * xa + ku[4] * xb + ku[5] * xc;
        ym[c] += ku[6] * xa + ku[7] * xb + ku[8] * xc;
      }
      for (int i = 0; i + 1 < n - j; ++i) {
        const int a = r0 + i + 1, b = r1 + i, c = r1 + i + 1;
        const double xa = xm[a], xb = xm[b], xc = xm[c];
        ym[a] += kd[0] * xa + kd[1] * xb + kd[2] * xc;
        ym[b] += kd[3] * xa + kd[4] * xb + kd[5] * xc;
        ym[c] += kd[6] * xa + kd[7] * xb + kd[8] * xc;
      }
    }
  }
  o2_interface_sync(h, l, y, 1);
}

/* for_each_lattice_boundary, proj/src/fem.cpp:53-58 + zero_domain_boundary :230-241 */
static void zero_domain_boundary(const oh2d* h, int l, double* f) {
  const int n = h->lev[l].n, S = h->lev[l].S;
  for (int s = 0; s < h->M; ++s) {
    double* fm = f + (size_t)s * S;
    for (int i = 0; i <= n; ++i)
      if (on_domain_boundary(h, s, l, i, 0)) fm[lat(n, i, 0)] = 0.0;
    for (int j = 1; j <= n; ++j)
      if (on_domain_boundary(h, s, l, 0, j)) fm[lat(n, 0, j)] = 0.0;
    for (int j = 1; j <= n - 1; ++j)
      if (on_domain_boundary(h, s, l, n - j, j)) fm[lat(n, n - j, j)] = 0.0;
  }
}

/* MultigridSolver::residual, proj/src/multigrid.cpp:183-190 */
void o2_residual(const oh2d* h, int l, const double* u, const double* b, double* r) {
  const size_t N = (size_t)h->M * h->lev[l].S;
  o2_apply(h, l, 0, u, r);
  for (size_t k = 0; k < N; ++k) r[k] *= -1.0;
  for (size_t k = 0; k < N; ++k) r[k] += 1.0 * b[k];
  zero_domain_boundary(h, l, r);
}

/* OperatorP1::partial_row, proj/src/fem.cpp:128-173 */
static void partial_row(const oh2d* h, int l, int slot, int i, int j, const double* x, double* diag, double* off) {
  const int n = h->lev[l].n;
  const double* ku = h->lev[l].ku + 9 * slot;
  const double* kd = h->lev[l].kd + 9 * slot;
  double d = 0.0, o = 0.0;
  if (i + j <= n - 1) { d += ku[0]; o += ku[1] * x[lat(n, i + 1, j)] + ku[2] * x[lat(n, i, j + 1)]; }
  if (i >= 1 && i - 1 + j <= n - 1) { d += ku[4]; o += ku[3] * x[lat(n, i - 1, j)] + ku[5] * x[lat(n, i - 1, j + 1)]; }
  if (j >= 1 && i + j - 1 <= n - 1) { d += ku[8]; o += ku[6] * x[lat(n, i, j - 1)] + ku[7] * x[lat(n, i + 1, j - 1)]; }
  if (i >= 1 && i + j <= n - 1) { d += kd[0]; o += kd[1] * x[lat(n, i - 1, j + 1)] + kd[2] * x[lat(n, i, j + 1)]; }
  if (j >= 1 && i + j <= n - 1) { d += kd[4]; o += kd[3] * x[lat(n, i + 1, j - 1)] + kd[5] * x[lat(n, i + 1, j)]; }
  if (i >= 1 && j >= 1 && i + j <= n) { d += kd[8]; o += kd[6] * x[lat(n, i, j - 1)] + kd[7] * x[lat(n, i - 1, j)]; }
  *diag = d;
  *off = o;
}

static void relax_boundary_node(const oh2d* h, int l, int slot, int i, int j, double* u, const double* b) {
  const o_level* lv = &h->lev[l];
  const int n = lv->n, S = lv->S;
  const int idx = lat(n, i, j);
  const int gid = boundary_group(h, slot, l, i, j);
  double value;
  if (on_domain_boundary(h, slot, l, i, j)) {
    value = b[(size_t)slot * S + idx];
  } else {
    double diag = 0.0, off = 0.0;
    for (int k = lv->gptr[gid]; k < lv->gptr[gid + 1]; ++k) {
      double d, o;
      partial_row(h, l, lv->mslot[k], lv->mi[k], lv->mj[k], u + (size_t)lv->mslot[k] * S, &d, &o);
      diag += d;
      off += o;
    }
    value = (b[(size_t)slot * S + idx] - off) / diag;
  }
  for (int k = lv->gptr[gid]; k < lv->gptr[gid + 1]; ++k) u[(size_t)lv->mslot[k] * S + lv->midx[k]] = value;
}

/* MultigridSolver::gauss_seidel, proj/src/multigrid.cpp:127-181 */
void o2_gauss_seidel(const oh2d* h, int l, double* u, const double* b, int sweeps) {
  const o_level* lv = &h->lev[l];
  const int n = lv->n, S = lv->S;
  for (int sw = 0; sw < sweeps; ++sw) {
    for (int slot = 0; slot < h->M; ++slot) {
      double* uu = u + (size_t)slot * S;
      const double* bb = b + (size_t)slot * S;
      const double* s = lv->st + 7 * slot;
      const double inv_c = 1.0 / s[0];
      for (int j = 0; j <= n; ++j) {
        const int row = lat(n, 0, j);
        const int imax = n - j;
        if (j == 0 || j == n) {
          for (int i = 0; i <= imax; ++i) relax_boundary_node(h, l, slot, i, j, u, b);
          continue;
        }
        relax_boundary_node(h, l, slot, 0, j, u, b);
        const int dn = n + 1 - j, dnw = n - j, ds = n + 2 - j, dse = n + 1 - j;
        for (int i = 1; i < imax; ++i) {
          const int k = row + i;
          const double acc = bb[k] - (s[1] * uu[k + 1] + s[2] * uu[k - 1] + s[3] * uu[k + dn] + s[4] * uu[k - ds] +
                                      s[5] * uu[k + dnw] + s[6] * uu[k - dse]);
          uu[k] = acc * inv_c;
        }
        if (imax >= 1) relax_boundary_node(h, l, slot, imax, j, u, b);
      }
    }
  }
}

/* prolongate, proj/src/multigrid.cpp:22-53 */
void o2_prolongate(const oh2d* h, int lc, const double* coarse, double* fine) {
  const int nc = h->lev[lc].n, nf = 2 * nc;
  const int Sc = h->lev[lc].S, Sf = latsize(nf);
  for (int s = 0; s < h->M; ++s) {
    const double* c = coarse + (size_t)s * Sc;
    double* f = fine + (size_t)s * Sf;
    for (int j = 0; j <= nf; ++j) {
      const int row = lat(nf, 0, j);
      for (int i = 0; i <= nf - j; ++i) {
        double v;
        if ((i & 1) == 0 && (j & 1) == 0) v = c[lat(nc, i / 2, j / 2)];
        else if ((j & 1) == 0) v = 0.5 * (c[lat(nc, (i - 1) / 2, j / 2)] + c[lat(nc, (i + 1) / 2, j / 2)]);
        else if ((i & 1) == 0) v = 0.5 * (c[lat(nc, i / 2, (j - 1) / 2)] + c[lat(nc, i / 2, (j + 1) / 2)]);
        else v = 0.5 * (c[lat(nc, (i + 1) / 2, (j - 1) / 2)] + c[lat(nc, (i - 1) / 2, (j + 1) / 2)]);
        f[row + i] = v;
      }
    }
  }
}

/* restrict_transpose, proj/src/multigrid.cpp:55-104 */
void o2_restrict(const oh2d* h, int lf, const double* fine, double* coarse) {
  const int lc = lf - 1;
  const int nc = h->lev[lc].n, nf = h->lev[lf].n;
  const int Sc = h->lev[lc].S, Sf = h->lev[lf].S;
  double* masked = (double*)malloc(sizeof(double) * (size_t)h->M * Sf);
  memcpy(masked, fine, sizeof(double) * (size_t)h->M * Sf);
  for (int s = 0; s < h->M; ++s) {
    double* m = masked + (size_t)s * Sf;
    for (int i = 0; i <= nf; ++i)
      if (!owns_boundary_node(h, s, lf, i, 0)) m[lat(nf, i, 0)] = 0.0;
    for (int j = 1; j <= nf; ++j)
      if (!owns_boundary_node(h, s, lf, 0, j)) m[lat(nf, 0, j)] = 0.0;
    for (int j = 1; j <= nf - 1; ++j)
      if (!owns_boundary_node(h, s, lf, nf - j, j)) m[lat(nf, nf - j, j)] = 0.0;
  }
  memset(coarse, 0, sizeof(double) * (size_t)h->M * Sc);
  for (int s = 0; s < h->M; ++s) {
    const double* f = masked + (size_t)s * Sf;
    double* c = coarse + (size_t)s * Sc;
    for (int j = 0; j <= nf; ++j) {
      const int row = lat(nf, 0, j);
      for (int i = 0; i <= nf - j; ++i) {
        const double v = f[row + i];
        if (v == 0.0) continue;
        if ((i & 1) == 0 && (j & 1) == 0) {
          c[lat(nc, i / 2, j / 2)] += v;
        } else if ((j & 1) == 0) {
          c[lat(nc, (i - 1) / 2, j / 2)] += 0.5 * v;
          c[lat(nc, (i + 1) / 2, j / 2)] += 0.5 * v;
        } else if ((i & 1) == 0) {
          c[lat(nc, i / 2, (j - 1) / 2)] += 0.5 * v;
          c[lat(nc, i / 2, (j + 1) / 2)] += 0.5 * v;
        } else {
          c[lat(nc, (i + 1) / 2, (j - 1) / 2)] += 0.5 * v;
          c[lat(nc, (i - 1) / 2, (j + 1) / 2)] += 0.5 * v;
        }
      }
    }
  }
  free(masked);
  o2_interface_sync(h, lc, coarse, 1);
}

/* MultigridSolver::cg_level0, proj/src/multigrid.cpp:198-229; returns 0 ok,
 * 1 not converged, 2 lost definiteness; *iters = iterations */
int o2_cg_level0(const oh2d* h, double* u, const double* b, double rel, double absf, int maxit, int* iters) {
  const size_t N = (size_t)h->M * h->lev[0].S;
  double* r = (double*)malloc(sizeof(double) * N);
  double* p = (double*)malloc(sizeof(double) * N);
  double* ap = (double*)malloc(sizeof(double) * N);
  double* bi = (double*)malloc(sizeof(double) * N);
  int status = 0, it = 0;
  o2_residual(h, 0, u, b, r);
  memcpy(p, r, sizeof(double) * N);
  double rr = o2_dot_unique(h, 0, r, r);
  memcpy(bi, b, sizeof(double) * N);
  zero_domain_boundary(h, 0, bi);
  const double bd = o2_dot_unique(h, 0, bi, bi);
  const double bnorm = sqrt(bd > 0.0 ? bd : 0.0);
  const double a = rel * bnorm;
  const double tol = a < absf ? absf : a;
  while (sqrt(rr) > tol) {
    if (++it > maxit) { status = 1; break; }
    o2_apply(h, 0, 0, p, ap);
    zero_domain_boundary(h, 0, ap);
    const double pap = o2_dot_unique(h, 0, p, ap);
    if (pap <= 0.0) { status = 2; break; }
    const double alpha = rr / pap;
    for (size_t k = 0; k < N; ++k) u[k] += alpha * p[k];
    for (size_t k = 0; k < N; ++k) r[k] += -alpha * ap[k];
    const double rr_new = o2_dot_unique(h, 0, r, r);
    const double beta = rr_new / rr;
    for (size_t k = 0; k < N; ++k) p[k] *= beta;
    for (size_t k = 0; k < N; ++k) p[k] += 1.0 * r[k];
    rr = rr_new;
  }
  if (iters) *iters = it;
  free(r); free(p); free(ap); free(bi);
  return status;
}

/* ---------------------------------------------------------------- problems */
static double f_sin(double x, double y) { return 2.0 * M_PI * M_PI * sin(M_PI * x) * sin(M_PI * y); }
static double u_sin(double x, double y) { return sin(M_PI * x) * sin(M_PI * y); }
static double zero2(double x, double y) { (void)x; (void)y; return 0.0; }
/* make_lshape_spec, proj/src/problems.cpp:36-53 */
static double u_lshape(double x, double y) {
  const double r = hypot(x, y);
  if (r == 0.0) return 0.0;
  double phi = atan2(y, x);
  if (phi < 0.0) phi += 2.0 * M_PI;
  return pow(r, 2.0 / 3.0) * sin(2.0 * phi / 3.0);
}

typedef double (*fn2)(double, double);

static void problem_fns(int kind, fn2* f, fn2* g) {
  if (kind == 1) { *f = f_sin; *g = u_sin; }
  else if (kind == 2) { *f = zero2; *g = u_lshape; }
  else { *f = zero2; *g = zero2; }
}

/* assemble_rhs, proj/src/fem.cpp:175-210 */
static void assemble_rhs(const oh2d* h, int l, fn2 f, double* bv) {
  const int n = h->lev[l].n, S = h->lev[l].S;
  memset(bv, 0, sizeof(double) * (size_t)h->M * S);
  for (int s = 0; s < h->M; ++s) {
    double* bm = bv + (size_t)s * S;
    const double cell_area = h->area[s] / ((double)n * n);
    const double w = cell_area / 3.0;
    const int* v = h->tri + 3 * s;
    const double c0x = h->vx[v[0]], c0y = h->vy[v[0]];
    const double ux = (h->vx[v[1]] - c0x) / n, uy = (h->vy[v[1]] - c0y) / n;
    const double wx = (h->vx[v[2]] - c0x) / n, wy = (h->vy[v[2]] - c0y) / n;
#define PX(i, j) (c0x + (i) * ux + (j) * wx)
#define PY(i, j) (c0y + (i) * uy + (j) * wy)
#define ADD_CELL(a, b_, c, i0, j0, i1, j1, i2, j2)                                          \
  do {                                                                                       \
    const double mi01 = 0.5 * ((double)(i0) + (double)(i1)), mj01 = 0.5 * ((double)(j0) + (double)(j1)); \
    const double mi02 = 0.5 * ((double)(i0) + (double)(i2)), mj02 = 0.5 * ((double)(j0) + (double)(j2)); \
    const double mi12 = 0.5 * ((double)(i1) + (double)(i2)), mj12 = 0.5 * ((double)(j1) + (double)(j2)); \
    const double f01 = f(PX(mi01, mj01), PY(mi01, mj01));                                   \
    const double f02 = f(PX(mi02, mj02), PY(mi02, mj02));                                   \
    const double f12 = f(PX(mi12, mj12), PY(mi12, mj12));                                   \
    bm[a] += w * 0.5 * (f01 + f02);                                                          \
    bm[b_] += w * 0.5 * (f01 + f12);                                                         \
    bm[c] += w * 0.5 * (f02 + f12);                                                          \
  } while (0)
    for (int j = 0; j < n; ++j) {
      const int r0 = lat(n, 0, j), r1 = lat(n, 0, j + 1);
      for (int i = 0; i < n - j; ++i) ADD_CELL(r0 + i, r0 + i + 1, r1 + i, i, j, i + 1, j, i, j + 1);
      for (int i = 0; i + 1 < n - j; ++i) ADD_CELL(r0 + i + 1, r1 + i, r1 + i + 1, i + 1, j, i, j + 1, i + 1, j + 1);
    }
#undef ADD_CELL
#undef PX
#undef PY
  }
  o2_interface_sync(h, l, bv, 1);
}

/* set_domain_boundary_values, proj/src/fem.cpp:212-228 */
static void set_domain_boundary_values(const oh2d* h, int l, double* fv, fn2 g) {
  const int n = h->lev[l].n, S = h->lev[l].S;
  for (int s = 0; s < h->M; ++s) {
    double* fm = fv + (size_t)s * S;
    double x, y;
    for (int i = 0; i <= n; ++i)
      if (on_domain_boundary(h, s, l, i, 0)) { node_xy(h, s, l, i, 0, &x, &y); fm[lat(n, i, 0)] = g(x, y); }
    for (int j = 1; j <= n; ++j)
      if (on_domain_boundary(h, s, l, 0, j)) { node_xy(h, s, l, 0, j, &x, &y); fm[lat(n, 0, j)] = g(x, y); }
    for (int j = 1; j <= n - 1; ++j)
      if (on_domain_boundary(h, s, l, n - j, j)) { node_xy(h, s, l, n - j, j, &x, &y); fm[lat(n, n - j, j)] = g(x, y); }
  }
  o2_interface_sync(h, l, fv, 0);
}

typedef struct {
  int pre, post;
  double rel, absf;
  int maxit;
  int status;
} o_cfg;

static void v_cycle(const oh2d* h, int l, double* u, const double* b, o_cfg* cfg) {
  if (l == 0) {
    int it;
    const int st = o2_cg_level0(h, u, b, cfg->rel, cfg->absf, cfg->maxit, &it);
    if (st && !cfg->status) cfg->status = st;
    return;
  }
  const size_t N = (size_t)h->M * h->lev[l].S, Nc = (size_t)h->M * h->lev[l - 1].S;
  o2_gauss_seidel(h, l, u, b, cfg->pre);
  double* r = (double*)malloc(sizeof(double) * N);
  double* rc = (double*)malloc(sizeof(double) * Nc);
  double* ec = (double*)calloc(Nc, sizeof(double));
  double* ef = (double*)malloc(sizeof(double) * N);
  o2_residual(h, l, u, b, r);
  o2_restrict(h, l, r, rc);
  zero_domain_boundary(h, l - 1, rc);
  v_cycle(h, l - 1, ec, rc, cfg);
  o2_prolongate(h, l - 1, ec, ef);
  for (size_t k = 0; k < N; ++k) u[k] += 1.0 * ef[k];
  o2_gauss_seidel(h, l, u, b, cfg->post);
  free(r); free(rc); free(ec); free(ef);
}

/* MultigridSolver::fmg with FinestPolicy::None, proj/src/multigrid.cpp:248-279.
 * u[l], b[l] (l = 0..L) and w[l] (l = 0..L-1, on level l+1) are caller-owned. */
int o2_fmg(const oh2d* h, int problem, int nu, int pre, int post, double rel, double absf, int maxit, double** u,
           double** b, double** w) {
  const int L = h->L;
  if (L < 1) return 3;
  fn2 f, g;
  problem_fns(problem, &f, &g);
  o_cfg cfg = {pre, post, rel, absf, maxit, 0};
  for (int l = 0; l <= L; ++l) {
    assemble_rhs(h, l, f, b[l]);
    set_domain_boundary_values(h, l, b[l], g);
  }
  memset(u[0], 0, sizeof(double) * (size_t)h->M * h->lev[0].S);
  set_domain_boundary_values(h, 0, u[0], g);
  {
    int it;
    const int st = o2_cg_level0(h, u[0], b[0], rel, absf, maxit, &it);
    if (st) cfg.status = st;
  }
  for (int l = 0; l < L; ++l) {
    o2_prolongate(h, l, u[l], w[l]);
    memcpy(u[l + 1], w[l], sizeof(double) * (size_t)h->M * h->lev[l + 1].S);
    set_domain_boundary_values(h, l + 1, u[l + 1], g);
    for (int c = 0; c < nu; ++c) v_cycle(h, l + 1, u[l + 1], b[l + 1], &cfg);
  }
  return cfg.status;
}

/* l2_norm / local_l2_norms, proj/src/fem.cpp:320-356 */
static double l2_norm(const oh2d* h, int l, const double* e) {
  const size_t N = (size_t)h->M * h->lev[l].S;
  double* me = (double*)malloc(sizeof(double) * N);
  o2_apply(h, l, 1, e, me);
  const double d = o2_dot_unique(h, l, e, me);
  free(me);
  return sqrt(d > 0.0 ? d : 0.0);
}

static void local_l2_norms(const oh2d* h, int l, const double* e, double* out) {
  const int n = h->lev[l].n, S = h->lev[l].S;
  for (int s = 0; s < h->M; ++s) {
    const double* fm = e + (size_t)s * S;
    const double* ku = h->lev[l].mu + 9 * s;
    const double* kd = h->lev[l].md + 9 * s;
    double sum = 0.0;
#define CELL(k, a, b, c)                                                                          \
  do {                                                                                            \
    const double xa = fm[a], xb = fm[b], xc = fm[c];                                              \
    sum += xa * (k[0] * xa + k[1] * xb + k[2] * xc) + xb * (k[3] * xa + k[4] * xb + k[5] * xc) +  \
           xc * (k[6] * xa + k[7] * xb + k[8] * xc);                                              \
  } while (0)
    for (int j = 0; j < n; ++j) {
      const int r0 = lat(n, 0, j), r1 = lat(n, 0, j + 1);
      for (int i = 0; i < n - j; ++i) CELL(ku, r0 + i, r0 + i + 1, r1 + i);
      for (int i = 0; i + 1 < n - j; ++i) CELL(kd, r0 + i + 1, r1 + i, r1 + i + 1);
    }
#undef CELL
    out[s] = sqrt(sum > 0.0 ? sum : 0.0);
  }
}

/* error_estimate, proj/src/estimator.cpp:8-45.  uL on level L, w[l] on level
 * l+1.  out4 = norm_base, norm_coarser, conv_factor, eta; returns 1 on a bad offset. */
int o2_estimate(const oh2d* h, const double* uL, double** w, int offset, int kind, double* out4, double* eta_local) {
  const int L = h->L;
  if (offset < 1 || offset > L - 1) return 1;
  const int base = L - offset;
  const size_t N = (size_t)h->M * h->lev[L].S;
  double* eb = (double*)malloc(sizeof(double) * N);
  double* ec = (double*)malloc(sizeof(double) * N);
  /* prolongate_to(w[base], L) and prolongate_to(w[base-1], L) */
  double* bufs[2] = {eb, ec};
  const int srcs[2] = {base, base - 1};
  for (int q = 0; q < 2; ++q) {
    int lv = srcs[q] + 1;
    double* cur = (double*)malloc(sizeof(double) * (size_t)h->M * h->lev[lv].S);
    memcpy(cur, w[srcs[q]], sizeof(double) * (size_t)h->M * h->lev[lv].S);
    while (lv < L) {
      double* nxt = (double*)malloc(sizeof(double) * (size_t)h->M * h->lev[lv + 1].S);
      o2_prolongate(h, lv, cur, nxt);
      free(cur);
      cur = nxt;
      ++lv;
    }
    for (size_t k = 0; k < N; ++k) bufs[q][k] = uL[k] + -1.0 * cur[k];
    free(cur);
  }
  const double nb = l2_norm(h, L, eb), nc = l2_norm(h, L, ec);
  const double conv = nc > 0.0 ? nb / nc : 0.0;
  out4[0] = nb;
  out4[1] = nc;
  out4[2] = conv;
  out4[3] = pow(conv, offset) * nb;
  double* lb = (double*)malloc(sizeof(double) * h->M);
  local_l2_norms(h, L, eb, lb);
  if (kind == 0) {
    memcpy(eta_local, lb, sizeof(double) * h->M);
  } else {
    double* lc = (double*)malloc(sizeof(double) * h->M);
    local_l2_norms(h, L, ec, lc);
    const double floor = 1e-14 * nc;
    for (int t = 0; t < h->M; ++t) {
      const double conv_t = lc[t] > floor ? lb[t] / lc[t] : conv;
      eta_local[t] = pow(conv_t, offset) * lb[t];
    }
    free(lc);
  }
  free(lb); free(eb); free(ec);
  return 0;
}
