/*
 * TEST INFRASTRUCTURE — CPU oracle of the 3-d hot path (configs 3-5).
 * Not product code: only tests/ and bench.py's CPU-baseline legs may load it.
 *
 * The reference has no 3-d solver (proj/src/hhg.cpp:49-50 throws for
 * dim != 2), so PARITY IS UNPINNED against the reference here: this file is
 * an independent plain-C restatement of the builder's 3-d specification
 * (DESIGN.md §3-d), written in the style of the 2-d reference:
 *   lattice / groups / ownership        like proj/src/hhg.cpp:48-144, 206-257
 *   element matrices, apply             like proj/src/fem.cpp:30-126
 *   partial rows                        like proj/src/fem.cpp:128-173
 *   Gauss-Seidel                        builder's order (boundary groups by colour, then every macro's interior plane by plane, four parity classes per plane)
 *   residual, transfers, CG, V-cycle,
 *   FMG (FinestPolicy::None)            like proj/src/multigrid.cpp:22-279
 *   estimator                           like proj/src/estimator.cpp:8-45
 * RHS: b = M f_I (nodal interpolant, owner coordinates) with Dirichlet rows g.
 * Sequential loops, no FMA contraction (built without -march / -ffast-math).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MAXL3 9

static const int KUHN[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
static const int STEP[3][3] = {{1, 0, 0}, {-1, 1, 0}, {0, -1, 1}};
static const int DIR[15][3] = {{0, 0, 0},  {1, 0, 0},  {-1, 0, 0}, {-1, 1, 0}, {1, -1, 0},
                               {0, -1, 1}, {0, 1, -1}, {0, 1, 0},  {0, -1, 0}, {-1, 0, 1},
                               {1, 0, -1}, {1, -1, 1}, {-1, 1, -1}, {0, 0, 1}, {0, 0, -1}};

static int tsz(int n) { return (n + 1) * (n + 2) * (n + 3) / 6; }
static int lat2(int n, int i, int j) { return j * (n + 1) - (j * (j - 1)) / 2 + i; }
static int lat3(int n, int i, int j, int k) { return tsz(n) - tsz(n - k) + lat2(n - k, i, j); }
static int inl(int n, int i, int j, int k) { return i >= 0 && j >= 0 && k >= 0 && i + j + k <= n; }
static void cvert(int ty, int r, int* d) {
  d[0] = d[1] = d[2] = 0;
  for (int q = 0; q < r; ++q)
    for (int a = 0; a < 3; ++a) d[a] += STEP[KUHN[ty][q]][a];
}
/* boundary signature of a lattice node: which of the faces i = 0, j = 0, k = 0, w0 = 0 it lies on */
static int sig_of(int n, int i, int j, int k) {
  return (i == 0) | ((j == 0) << 1) | ((k == 0) << 2) | ((i + j + k == n) << 3);
}
static int dirix(int a, int b, int c) {
  for (int d = 0; d < 15; ++d)
    if (DIR[d][0] == a && DIR[d][1] == b && DIR[d][2] == c) return d;
  return -1;
}

typedef struct {
  int n, S;
  long long dofs;
  int ng;
  int *gptr, *mslot, *midx, *mi, *mj, *mk;
  unsigned char *gdom;
  int *gcol;
  double *gdiag;
  int *ncol;       /* per copy: colour */
  int *gid;        /* per copy: group or -1 */
  unsigned char *flag; /* bit0 boundary, bit1 domain, bit2 owner */
  double *K, *Mm;  /* 96 per macro */
  double *stK, *stM; /* 15 per macro */
  double *psK, *psM; /* partial stencils of lattice-boundary nodes: 16 signatures x 15 per macro */
  double *gx, *gy, *gz; /* per copy: node coordinates (owner's for shared nodes) */
} o3lev;

typedef struct {
  int M, L, C, nv;
  int *tet;  /* 4 per macro */
  double *xyz;
  o3lev lv[MAXL3 + 1];
} o3h;

static double det3(const double* a, const double* b, const double* c) {
  return a[0] * (b[1] * c[2] - b[2] * c[1]) - a[1] * (b[0] * c[2] - b[2] * c[0]) + a[2] * (b[0] * c[1] - b[1] * c[0]);
}

static void tetmat(double p[4][3], double* K, double* Mm) {
  double e[3][3], g[4][3];
  for (int r = 0; r < 3; ++r)
    for (int d = 0; d < 3; ++d) e[r][d] = p[r + 1][d] - p[0][d];
  const double det = det3(e[0], e[1], e[2]);
  const double vol = fabs(det) / 6.0;
  for (int a = 0; a < 3; ++a) {
    const double* u = e[(a + 1) % 3];
    const double* v = e[(a + 2) % 3];
    const double c[3] = {u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2], u[0] * v[1] - u[1] * v[0]};
    for (int d = 0; d < 3; ++d) g[a + 1][d] = c[d] / det;
  }
  for (int d = 0; d < 3; ++d) g[0][d] = -(g[1][d] + g[2][d] + g[3][d]);
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b) {
      K[4 * a + b] = vol * (g[a][0] * g[b][0] + g[a][1] * g[b][1] + g[a][2] * g[b][2]);
      Mm[4 * a + b] = (a == b ? vol / 10.0 : vol / 20.0);
    }
}

/* ---------------- primitives (sorted arrays + binary search) */
typedef struct { int a, b; } e2;
typedef struct { int a, b, c; } f3;
static int cmpe(const void* x, const void* y) {
  const e2 *p = x, *q = y;
  return p->a != q->a ? (p->a < q->a ? -1 : 1) : (p->b < q->b ? -1 : (p->b > q->b));
}
static int cmpf(const void* x, const void* y) {
  const f3 *p = x, *q = y;
  if (p->a != q->a) return p->a < q->a ? -1 : 1;
  if (p->b != q->b) return p->b < q->b ? -1 : 1;
  return p->c < q->c ? -1 : (p->c > q->c);
}
static void s3(int* v) {
  for (int a = 0; a < 3; ++a)
    for (int b = a + 1; b < 3; ++b)
      if (v[b] < v[a]) { int t = v[a]; v[a] = v[b]; v[b] = t; }
}

void o3_free(o3h* h) {
  if (!h) return;
  for (int l = 0; l <= h->L; ++l) {
    o3lev* v = &h->lv[l];
    free(v->gptr); free(v->mslot); free(v->midx); free(v->mi); free(v->mj); free(v->mk);
    free(v->gdom); free(v->gcol); free(v->gdiag); free(v->ncol); free(v->gid); free(v->flag);
    free(v->K); free(v->Mm); free(v->stK); free(v->stM); free(v->gx); free(v->gy); free(v->gz);
    free(v->psK); free(v->psM);
  }
  free(h->tet); free(h->xyz); free(h);
}

int o3_num_macros(const o3h* h) { return h->M; }
int o3_level_size(const o3h* h, int l) { return h->M * h->lv[l].S; }
long long o3_dofs(const o3h* h, int l) { return h->lv[l].dofs; }
int o3_colors(const o3h* h) { return h->C; }

o3h* o3_build(int nv, const double* xyz, int ne, const int* tet_in, int L) {
  if (nv <= 0 || ne <= 0 || L < 0 || L > MAXL3) return NULL;
  o3h* h = calloc(1, sizeof(o3h));
  h->M = ne; h->L = L; h->nv = nv;
  h->xyz = malloc(sizeof(double) * 3 * nv);
  memcpy(h->xyz, xyz, sizeof(double) * 3 * nv);
  h->tet = malloc(sizeof(int) * 4 * ne);
  for (int s = 0; s < ne; ++s) {
    int* t = &h->tet[4 * s];
    for (int q = 0; q < 4; ++q) t[q] = tet_in[4 * s + q];
    double a[3], b[3], c[3];
    for (int d = 0; d < 3; ++d) {
      a[d] = xyz[3 * t[1] + d] - xyz[3 * t[0] + d];
      b[d] = xyz[3 * t[2] + d] - xyz[3 * t[0] + d];
      c[d] = xyz[3 * t[3] + d] - xyz[3 * t[0] + d];
    }
    if (det3(a, b, c) < 0.0) { int tmp = t[2]; t[2] = t[3]; t[3] = tmp; }
  }
  /* edges, faces */
  e2* E = malloc(sizeof(e2) * 6 * ne);
  f3* F = malloc(sizeof(f3) * 4 * ne);
  int nE = 0, nF = 0;
  for (int s = 0; s < ne; ++s) {
    const int* t = &h->tet[4 * s];
    for (int a = 0; a < 4; ++a)
      for (int b = a + 1; b < 4; ++b) {
        E[nE].a = t[a] < t[b] ? t[a] : t[b];
        E[nE].b = t[a] < t[b] ? t[b] : t[a];
        ++nE;
      }
    for (int o = 0; o < 4; ++o) {
      int v[3], q = 0;
      for (int a = 0; a < 4; ++a)
        if (a != o) v[q++] = t[a];
      s3(v);
      F[nF].a = v[0]; F[nF].b = v[1]; F[nF].c = v[2];
      ++nF;
    }
  }
  qsort(E, nE, sizeof(e2), cmpe);
  qsort(F, nF, sizeof(f3), cmpf);
  int ue = 0, uf = 0;
  int* fuse = calloc(nF, sizeof(int));
  for (int q = 0; q < nE; ++q)
    if (q == 0 || cmpe(&E[q], &E[ue - 1])) E[ue++] = E[q];
  for (int q = 0; q < nF; ++q) {
    if (q == 0 || cmpf(&F[q], &F[uf - 1])) { F[uf] = F[q]; fuse[uf] = 0; ++uf; }
    ++fuse[uf - 1];
  }
  nE = ue; nF = uf;
  /* domain boundary of vertices / edges */
  unsigned char* vb = calloc(nv, 1);
  unsigned char* eb = calloc(nE, 1);
  for (int f = 0; f < nF; ++f)
    if (fuse[f] == 1) {
      vb[F[f].a] = vb[F[f].b] = vb[F[f].c] = 1;
      const e2 ks[3] = {{F[f].a, F[f].b}, {F[f].a, F[f].c}, {F[f].b, F[f].c}};
      for (int q = 0; q < 3; ++q) {
        e2* hit = bsearch(&ks[q], E, nE, sizeof(e2), cmpe);
        eb[hit - E] = 1;
      }
    }
  /* vertex colouring: grid parity (Kuhn meshes) else greedy with the tet-XOR rule */
  int* vc = calloc(nv, sizeof(int));
  {
    double hmin = 1e300, mn[3] = {1e300, 1e300, 1e300};
    for (int v = 0; v < nv; ++v)
      for (int d = 0; d < 3; ++d)
        if (xyz[3 * v + d] < mn[d]) mn[d] = xyz[3 * v + d];
    for (int q = 0; q < nE; ++q) {
      double m = 0.0;
      for (int d = 0; d < 3; ++d) {
        const double df = fabs(xyz[3 * E[q].a + d] - xyz[3 * E[q].b + d]);
        if (df > m) m = df;
      }
      if (m < hmin) hmin = m;
    }
    int grid = hmin > 0.0;
    for (int v = 0; v < nv && grid; ++v) {
      int c = 0;
      for (int d = 0; d < 3; ++d) {
        const double qd = (xyz[3 * v + d] - mn[d]) / hmin, r = round(qd);
        if (fabs(qd - r) > 1e-9) grid = 0;
        c |= (int)(((long long)r) & 1) << d;
      }
      vc[v] = c;
    }
    for (int s = 0; s < ne && grid; ++s) {
      const int* t = &h->tet[4 * s];
      for (int a = 0; a < 4; ++a)
        for (int b = a + 1; b < 4; ++b)
          if (vc[t[a]] == vc[t[b]]) grid = 0;
      if ((vc[t[0]] ^ vc[t[1]] ^ vc[t[2]] ^ vc[t[3]]) == 0) grid = 0;
    }
    if (grid) {
      h->C = 8;
    } else {
      int mx = 0;
      for (int v = 0; v < nv; ++v) {
        int c = 0, ok = 0;
        while (!ok) {
          ok = 1;
          for (int s = 0; s < ne && ok; ++s) {
            const int* t = &h->tet[4 * s];
            int has = 0, lower = 1, x = c;
            for (int a = 0; a < 4; ++a) {
              if (t[a] == v) has = 1;
              else if (t[a] > v) lower = 0;
            }
            if (!has) continue;
            for (int a = 0; a < 4; ++a)
              if (t[a] < v && vc[t[a]] == c) ok = 0;
            if (ok && lower) {
              for (int a = 0; a < 4; ++a)
                if (t[a] != v) x ^= vc[t[a]];
              if (x == 0) ok = 0;
            }
          }
          if (!ok) ++c;
        }
        vc[v] = c;
        if (c > mx) mx = c;
      }
      h->C = 2;
      while (h->C < mx + 1) h->C <<= 1;
    }
  }
  for (int l = 0; l <= L; ++l) {
    o3lev* lv = &h->lv[l];
    const int n = 1 << l, S = tsz(n);
    (void)0;
    lv->n = n; lv->S = S;
    const long long pf = n >= 3 ? (long long)(n - 1) * (n - 2) / 2 : 0;
    const int ng = (int)(nv + (long long)nE * (n - 1) + nF * pf);
    lv->ng = ng;
    lv->gid = malloc(sizeof(int) * (size_t)ne * S);
    lv->flag = calloc((size_t)ne * S, 1);
    lv->ncol = malloc(sizeof(int) * (size_t)ne * S);
    int* cnt = calloc(ng + 1, sizeof(int));
    for (int pass = 0; pass < 2; ++pass) {
      int* fillp = NULL;
      if (pass == 1) {
        for (int g = 0; g < ng; ++g) cnt[g + 1] += cnt[g];
        lv->gptr = malloc(sizeof(int) * (ng + 1));
        memcpy(lv->gptr, cnt, sizeof(int) * (ng + 1));
        const int nm = cnt[ng];
        lv->mslot = malloc(sizeof(int) * nm); lv->midx = malloc(sizeof(int) * nm);
        lv->mi = malloc(sizeof(int) * nm); lv->mj = malloc(sizeof(int) * nm); lv->mk = malloc(sizeof(int) * nm);
        lv->gdom = calloc(ng, 1); lv->gcol = calloc(ng, sizeof(int));
        fillp = malloc(sizeof(int) * ng);
        memcpy(fillp, cnt, sizeof(int) * ng);
      }
      for (int s = 0; s < ne; ++s) {
        const int* t = &h->tet[4 * s];
        for (int k = 0; k <= n; ++k)
          for (int j = 0; j <= n - k; ++j)
            for (int i = 0; i <= n - k - j; ++i) {
              const int w[4] = {n - i - j - k, i, j, k};
              const size_t off = (size_t)s * S + lat3(n, i, j, k);
              int col = 0;
              for (int q = 0; q < 4; ++q)
                if (w[q] & 1) col ^= vc[t[q]];
              lv->ncol[off] = col;
              if (w[0] > 0 && i > 0 && j > 0 && k > 0) { lv->gid[off] = -1; continue; }
              int sv[4], sw[4], c = 0;
              for (int q = 0; q < 4; ++q)
                if (w[q] > 0) { sv[c] = t[q]; sw[c] = w[q]; ++c; }
              for (int a = 0; a < c; ++a)
                for (int b = a + 1; b < c; ++b)
                  if (sv[b] < sv[a]) {
                    int x = sv[a]; sv[a] = sv[b]; sv[b] = x;
                    x = sw[a]; sw[a] = sw[b]; sw[b] = x;
                  }
              int g, dom;
              if (c == 1) { g = sv[0]; dom = vb[sv[0]]; }
              else if (c == 2) {
                e2 key = {sv[0], sv[1]};
                const int ei = (int)((e2*)bsearch(&key, E, nE, sizeof(e2), cmpe) - E);
                g = nv + ei * (n - 1) + (sw[1] - 1);
                dom = eb[ei];
              } else {
                f3 key = {sv[0], sv[1], sv[2]};
                const int fi = (int)((f3*)bsearch(&key, F, nF, sizeof(f3), cmpf) - F);
                g = (int)(nv + (long long)nE * (n - 1) + fi * pf + lat2(n - 3, sw[1] - 1, sw[2] - 1));
                dom = fuse[fi] == 1;
              }
              lv->gid[off] = g;
              if (pass == 0) { ++cnt[g + 1]; continue; }
              const int slot = fillp[g]++;
              lv->mslot[slot] = s; lv->midx[slot] = lat3(n, i, j, k);
              lv->mi[slot] = i; lv->mj[slot] = j; lv->mk[slot] = k;
              lv->gdom[g] = (unsigned char)dom;
              lv->gcol[g] = col;
              lv->flag[off] = (unsigned char)(1 | (dom ? 2 : 0) | (slot == lv->gptr[g] ? 4 : 0));
            }
      }
      free(fillp);
    }
    free(cnt);
    const long long inter = n >= 4 ? (long long)(n - 1) * (n - 2) * (n - 3) / 6 : 0;
    lv->dofs = nv + (long long)nE * (n - 1) + nF * pf + (long long)ne * inter;
    /* element matrices and stencils */
    lv->K = calloc(96 * (size_t)ne, sizeof(double)); lv->Mm = calloc(96 * (size_t)ne, sizeof(double));
    lv->stK = calloc(15 * (size_t)ne, sizeof(double)); lv->stM = calloc(15 * (size_t)ne, sizeof(double));
    for (int s = 0; s < ne; ++s) {
      const int* t = &h->tet[4 * s];
      for (int ty = 0; ty < 6; ++ty) {
        double p[4][3];
        for (int r = 0; r < 4; ++r) {
          int d[3];
          cvert(ty, r, d);
          for (int a = 0; a < 3; ++a)
            p[r][a] = xyz[3 * t[0] + a] + ((double)d[0] / n) * (xyz[3 * t[1] + a] - xyz[3 * t[0] + a]) +
                      ((double)d[1] / n) * (xyz[3 * t[2] + a] - xyz[3 * t[0] + a]) +
                      ((double)d[2] / n) * (xyz[3 * t[3] + a] - xyz[3 * t[0] + a]);
        }
        tetmat(p, &lv->K[96 * s + 16 * ty], &lv->Mm[96 * s + 16 * ty]);
      }
      for (int ty = 0; ty < 6; ++ty)
        for (int r = 0; r < 4; ++r)
          for (int c = 0; c < 4; ++c) {
            int dr[3], dc[3];
            cvert(ty, r, dr); cvert(ty, c, dc);
            const int d = dirix(dc[0] - dr[0], dc[1] - dr[1], dc[2] - dr[2]);
            lv->stK[15 * s + d] += lv->K[96 * s + 16 * ty + 4 * r + c];
            lv->stM[15 * s + d] += lv->Mm[96 * s + 16 * ty + 4 * r + c];
          }
    }
    /* partial stencils: for every signature, from the first node (lattice order)
     * carrying it, the sum over its existing cells (type, role, column order) */
    lv->psK = calloc(240 * (size_t)ne, sizeof(double));
    lv->psM = calloc(240 * (size_t)ne, sizeof(double));
    for (int s = 0; s < ne; ++s) {
      int done = 0;
      for (int k = 0; k <= n; ++k)
        for (int j = 0; j <= n - k; ++j)
          for (int i = 0; i <= n - k - j; ++i) {
            const int sg = sig_of(n, i, j, k);
            if (sg == 0 || ((done >> sg) & 1)) continue;
            done |= 1 << sg;
            double* pk = lv->psK + 240 * (size_t)s + 15 * sg;
            double* pm = lv->psM + 240 * (size_t)s + 15 * sg;
            for (int ty = 0; ty < 6; ++ty)
              for (int r = 0; r < 4; ++r) {
                int dr[3], ok = 1;
                cvert(ty, r, dr);
                for (int c = 0; c < 4 && ok; ++c) {
                  int dc[3];
                  cvert(ty, c, dc);
                  ok = inl(n, i - dr[0] + dc[0], j - dr[1] + dc[1], k - dr[2] + dc[2]);
                }
                if (!ok) continue;
                for (int c = 0; c < 4; ++c) {
                  int dc[3];
                  cvert(ty, c, dc);
                  const int d = dirix(dc[0] - dr[0], dc[1] - dr[1], dc[2] - dr[2]);
                  pk[d] += lv->K[96 * s + 16 * ty + 4 * r + c];
                  pm[d] += lv->Mm[96 * s + 16 * ty + 4 * r + c];
                }
              }
          }
    }
    /* group diagonals */
    lv->gdiag = calloc(ng, sizeof(double));
    for (int g = 0; g < ng; ++g) {
      double diag = 0.0;
      for (int q = lv->gptr[g]; q < lv->gptr[g + 1]; ++q)
        diag += lv->psK[240 * (size_t)lv->mslot[q] + 15 * sig_of(n, lv->mi[q], lv->mj[q], lv->mk[q])];
      lv->gdiag[g] = diag;
    }
    /* node coordinates, shared nodes from their owner */
    lv->gx = malloc(sizeof(double) * (size_t)ne * S);
    lv->gy = malloc(sizeof(double) * (size_t)ne * S);
    lv->gz = malloc(sizeof(double) * (size_t)ne * S);
    for (int s = 0; s < ne; ++s) {
      for (int k = 0; k <= n; ++k)
        for (int j = 0; j <= n - k; ++j)
          for (int i = 0; i <= n - k - j; ++i) {
            const size_t off = (size_t)s * S + lat3(n, i, j, k);
            int os = s, oi = i, oj = j, ok = k;
            if (lv->gid[off] >= 0) {
              const int f = lv->gptr[lv->gid[off]];
              os = lv->mslot[f]; oi = lv->mi[f]; oj = lv->mj[f]; ok = lv->mk[f];
            }
            const int* to = &h->tet[4 * os];
            double p[3];
            for (int a = 0; a < 3; ++a)
              p[a] = xyz[3 * to[0] + a] + ((double)oi / n) * (xyz[3 * to[1] + a] - xyz[3 * to[0] + a]) +
                     ((double)oj / n) * (xyz[3 * to[2] + a] - xyz[3 * to[0] + a]) +
                     ((double)ok / n) * (xyz[3 * to[3] + a] - xyz[3 * to[0] + a]);
            lv->gx[off] = p[0]; lv->gy[off] = p[1]; lv->gz[off] = p[2];
          }
    }
  }
  free(E); free(F); free(fuse); free(vb); free(eb); free(vc);
  return h;
}

/* ---------------- operators */
/* partial row of lattice-boundary node (i,j,k) of macro s: its signature's
 * partial stencil over the neighbours inside the macro, centre first */
static double partial_full(const o3lev* lv, const double* ps_all, int s, int i, int j, int k, const double* x) {
  const int n = lv->n;
  const double* xm = x + (size_t)s * lv->S;
  const double* ps = ps_all + 240 * (size_t)s + 15 * sig_of(n, i, j, k);
  double acc = ps[0] * xm[lat3(n, i, j, k)];
  for (int d = 1; d < 15; ++d) {
    const int a = i + DIR[d][0], b = j + DIR[d][1], c = k + DIR[d][2];
    if (inl(n, a, b, c)) acc = acc + ps[d] * xm[lat3(n, a, b, c)];
  }
  return acc;
}
/* off-diagonal part (Gauss-Seidel) */
static double partial_off(const o3lev* lv, int s, int i, int j, int k, const double* x) {
  const int n = lv->n;
  const double* xm = x + (size_t)s * lv->S;
  const double* ps = lv->psK + 240 * (size_t)s + 15 * sig_of(n, i, j, k);
  double o = 0.0;
  for (int d = 1; d < 15; ++d) {
    const int a = i + DIR[d][0], b = j + DIR[d][1], c = k + DIR[d][2];
    if (inl(n, a, b, c)) o = o + ps[d] * xm[lat3(n, a, b, c)];
  }
  return o;
}
static double stencil_apply(const o3lev* lv, const double* st, int s, int i, int j, int k, const double* x,
                            int skip_centre) {
  const int n = lv->n;
  const double* xm = x + (size_t)s * lv->S;
  double acc;
  int d0;
  if (skip_centre) {
    acc = st[1] * xm[lat3(n, i + DIR[1][0], j + DIR[1][1], k + DIR[1][2])];
    d0 = 2;
  } else {
    acc = st[0] * xm[lat3(n, i, j, k)];
    d0 = 1;
  }
  for (int d = d0; d < 15; ++d) acc = acc + st[d] * xm[lat3(n, i + DIR[d][0], j + DIR[d][1], k + DIR[d][2])];
  return acc;
}

/* y = Op x (mass = 0 stiffness, 1 mass), additive interface sync */
void o3_apply(const o3h* h, int l, int mass, const double* x, double* y) {
  const o3lev* lv = &h->lv[l];
  const int n = lv->n, S = lv->S;
  const double* Kt = mass ? lv->psM : lv->psK;
  const double* stt = mass ? lv->stM : lv->stK;
  for (int s = 0; s < h->M; ++s)
    for (int k = 1; k <= n; ++k)
      for (int j = 1; j <= n - k; ++j)
        for (int i = 1; i <= n - k - j; ++i)
          if (n - i - j - k > 0) y[(size_t)s * S + lat3(n, i, j, k)] = stencil_apply(lv, stt + 15 * s, s, i, j, k, x, 0);
  for (int g = 0; g < lv->ng; ++g) {
    const int b = lv->gptr[g], e = lv->gptr[g + 1];
    double v;
    if (e - b == 1) v = partial_full(lv, Kt, lv->mslot[b], lv->mi[b], lv->mj[b], lv->mk[b], x);
    else {
      v = 0.0;
      for (int q = b; q < e; ++q) v += partial_full(lv, Kt, lv->mslot[q], lv->mi[q], lv->mj[q], lv->mk[q], x);
    }
    for (int q = b; q < e; ++q) y[(size_t)lv->mslot[q] * S + lv->midx[q]] = v;
  }
}

/* r = b - A u, zero on domain-boundary copies */
void o3_residual(const o3h* h, int l, const double* u, const double* b, double* r) {
  const o3lev* lv = &h->lv[l];
  const size_t N = (size_t)h->M * lv->S;
  o3_apply(h, l, 0, u, r);
  for (size_t q = 0; q < N; ++q) r[q] = (lv->flag[q] & 2) ? 0.0 : b[q] - r[q];
}

/* Gauss-Seidel: boundary groups by colour, then the macro interiors plane by plane */
void o3_gauss_seidel(const o3h* h, int l, double* u, const double* b, int sweeps) {
  const o3lev* lv = &h->lv[l];
  const int n = lv->n, S = lv->S;
  for (int sw = 0; sw < sweeps; ++sw) {
    for (int c = 0; c < h->C; ++c)
      for (int g = 0; g < lv->ng; ++g) {
        if (lv->gcol[g] != c) continue;
        const int bq = lv->gptr[g], e = lv->gptr[g + 1];
        const size_t own = (size_t)lv->mslot[bq] * S + lv->midx[bq];
        double val;
        if (lv->gdom[g]) {
          val = b[own];
        } else {
          double off = 0.0;
          for (int q = bq; q < e; ++q) off = off + partial_off(lv, lv->mslot[q], lv->mi[q], lv->mj[q], lv->mk[q], u);
          val = (b[own] - off) / lv->gdiag[g];
        }
        for (int q = bq; q < e; ++q) u[(size_t)lv->mslot[q] * S + lv->midx[q]] = val;
      }
    /* interiors: every macro plane by plane (k ascending); inside a plane the
     * four (i, j) parity classes in the order (odd, odd), (even, odd),
     * (odd, even), (even, even) — nodes of one class are never neighbours.
     * The row is two fused chains (directions 1..7 and 8..14), added last. */
    for (int s = 0; s < h->M; ++s) {
      const double* st = lv->stK + 15 * s;
      const double inv_c = 1.0 / st[0];
      double* um = u + (size_t)s * S;
      for (int k = 1; k <= n - 3; ++k)
        for (int q = 0; q < 4; ++q)
          for (int j = 1 + (q >> 1); j <= n - 2 - k; j += 2)
            for (int i = 1 + (q & 1); i <= n - 1 - k - j; i += 2) {
              double x[15];
              for (int d = 1; d < 15; ++d) x[d] = um[lat3(n, i + DIR[d][0], j + DIR[d][1], k + DIR[d][2])];
              double a0 = st[1] * x[1], a1 = st[8] * x[8];
              for (int d = 2; d < 8; ++d) a0 = fma(st[d], x[d], a0);
              for (int d = 9; d < 15; ++d) a1 = fma(st[d], x[d], a1);
              const size_t off = (size_t)s * S + lat3(n, i, j, k);
              u[off] = (b[off] - (a0 + a1)) * inv_c;
            }
    }
  }
}

/* linear interpolation coarse level lc -> lc + 1 (per macro, no sync) */
static const int PDIR[8] = {-1, 1, 7, 3, 13, 9, 5, 11}; /* parity pattern -> direction index */
void o3_prolongate(const o3h* h, int lc, const double* c, double* f) {
  const o3lev* cv = &h->lv[lc];
  const o3lev* fv = &h->lv[lc + 1];
  const int nf = fv->n, nc = cv->n;
  for (int s = 0; s < h->M; ++s)
    for (int k = 0; k <= nf; ++k)
      for (int j = 0; j <= nf - k; ++j)
        for (int i = 0; i <= nf - k - j; ++i) {
          const int p = (i & 1) | ((j & 1) << 1) | ((k & 1) << 2);
          const double* cm = c + (size_t)s * cv->S;
          double v;
          if (p == 0) v = cm[lat3(nc, i / 2, j / 2, k / 2)];
          else {
            const int* d = DIR[PDIR[p]];
            const int ai = (i - d[0]) / 2, aj = (j - d[1]) / 2, ak = (k - d[2]) / 2;
            const int bi = (i + d[0]) / 2, bj = (j + d[1]) / 2, bk = (k + d[2]) / 2;
            v = 0.5 * (cm[lat3(nc, ai, aj, ak)] + cm[lat3(nc, bi, bj, bk)]);
          }
          f[(size_t)s * fv->S + lat3(nf, i, j, k)] = v;
        }
}

/* transpose: non-owner copies masked, fine visit order 0..14, additive coarse sync */
void o3_restrict(const o3h* h, int lf, const double* f, double* c) {
  const o3lev* fv = &h->lv[lf];
  const o3lev* cv = &h->lv[lf - 1];
  const int nf = fv->n, nc = cv->n;
  for (int s = 0; s < h->M; ++s) {
    const double* fm = f + (size_t)s * fv->S;
    const unsigned char* fl = fv->flag + (size_t)s * fv->S;
    for (int k = 0; k <= nc; ++k)
      for (int j = 0; j <= nc - k; ++j)
        for (int i = 0; i <= nc - k - j; ++i) {
          double acc = 0.0;
          for (int d = 0; d < 15; ++d) {
            const int a = 2 * i + DIR[d][0], b = 2 * j + DIR[d][1], cc = 2 * k + DIR[d][2];
            if (!inl(nf, a, b, cc)) continue;
            const int idx = lat3(nf, a, b, cc);
            const double v = (fl[idx] & 1) && !(fl[idx] & 4) ? 0.0 : fm[idx];
            acc = acc + (d == 0 ? v : 0.5 * v);
          }
          c[(size_t)s * cv->S + lat3(nc, i, j, k)] = acc;
        }
  }
  for (int g = 0; g < cv->ng; ++g) {
    const int b = cv->gptr[g], e = cv->gptr[g + 1];
    if (e - b < 2) continue;
    double v = 0.0;
    for (int q = b; q < e; ++q) v += c[(size_t)cv->mslot[q] * cv->S + cv->midx[q]];
    for (int q = b; q < e; ++q) c[(size_t)cv->mslot[q] * cv->S + cv->midx[q]] = v;
  }
}

/* owner inner product: the terms -- groups in order (owner copy), then the
 * interior nodes per macro in lattice order -- summed in chunks of 32
 * consecutive terms (sequentially), then the chunk sums sequentially */
typedef struct { double total, chunk; int count; } o3acc;
static void acc_add(o3acc* a, double t) {
  a->chunk += t;
  if (++a->count == 32) { a->total += a->chunk; a->chunk = 0.0; a->count = 0; }
}
double o3_dot(const o3h* h, int l, const double* a, const double* b) {
  const o3lev* lv = &h->lv[l];
  const int n = lv->n, S = lv->S;
  o3acc acc = {0.0, 0.0, 0};
  for (int g = 0; g < lv->ng; ++g) {
    const size_t o = (size_t)lv->mslot[lv->gptr[g]] * S + lv->midx[lv->gptr[g]];
    acc_add(&acc, a[o] * b[o]);
  }
  for (int m = 0; m < h->M; ++m)
    for (int k = 1; k <= n; ++k)
      for (int j = 1; j <= n - k; ++j)
        for (int i = 1; i <= n - k - j; ++i)
          if (n - i - j - k > 0) {
            const size_t o = (size_t)m * S + lat3(n, i, j, k);
            acc_add(&acc, a[o] * b[o]);
          }
  if (acc.count) acc.total += acc.chunk;
  return acc.total;
}

/* ---------------- problems (host glibc), RHS */
typedef double (*o3fn)(double, double, double, const double*);
static double sin3(double x, double y, double z, const double* p) {
  (void)p;
  return sin(M_PI * x) * sin(M_PI * y) * sin(M_PI * z);
}
static double sin3_f(double x, double y, double z, const double* p) { return 3.0 * M_PI * M_PI * sin3(x, y, z, p); }
static double gauss3(double x, double y, double z, const double* p) {
  (void)p;
  const double dx = x - 0.5, dy = y - 0.5, dz = z - 0.5;
  return exp(-1000.0 * (dx * dx + dy * dy + dz * dz));
}
static double gauss3_f(double x, double y, double z, const double* p) {
  const double dx = x - 0.5, dy = y - 0.5, dz = z - 0.5, r2 = dx * dx + dy * dy + dz * dz;
  return (6.0 * 1000.0 - 4.0 * 1000.0 * 1000.0 * r2) * gauss3(x, y, z, p);
}
/* sine series: p[0..63] = C_abc (a, b, c = 1..4, a fastest) */
/* acc += C_abc * ((sin(a pi x) * sin(b pi y)) * sin(c pi z)) in (c, b, a) order; the
 * twelve sines are formed once per point (the same values, so the same bits
 * as evaluating them inside the sum) */
static double series_f(double x, double y, double z, const double* p) {
  double sx[5], sy[5], sz[5];
  for (int a = 1; a <= 4; ++a) {
    sx[a] = sin(a * M_PI * x);
    sy[a] = sin(a * M_PI * y);
    sz[a] = sin(a * M_PI * z);
  }
  double acc = 0.0;
  for (int c = 1; c <= 4; ++c)
    for (int b = 1; b <= 4; ++b)
      for (int a = 1; a <= 4; ++a) acc += p[(a - 1) + 4 * (b - 1) + 16 * (c - 1)] * (sx[a] * sy[b] * sz[c]);
  return acc;
}
static double zero3(double x, double y, double z, const double* p) {
  (void)x; (void)y; (void)z; (void)p;
  return 0.0;
}
/* problem 0 zero, 1 sin3 (cfg3), 2 gauss (cfg4), 3 series with g = 0 (cfg5) */
static void pick(int prob, o3fn* f, o3fn* g) {
  *f = prob == 1 ? sin3_f : prob == 2 ? gauss3_f : prob == 3 ? series_f : zero3;
  *g = prob == 1 ? sin3 : prob == 2 ? gauss3 : zero3;
}

void o3_rhs(const o3h* h, int l, int prob, const double* par, double* b) {
  const o3lev* lv = &h->lv[l];
  const size_t N = (size_t)h->M * lv->S;
  o3fn f, g;
  pick(prob, &f, &g);
  double* fi = malloc(sizeof(double) * N);
  for (size_t q = 0; q < N; ++q) fi[q] = f(lv->gx[q], lv->gy[q], lv->gz[q], par);
  o3_apply(h, l, 1, fi, b);
  for (size_t q = 0; q < N; ++q)
    if (lv->flag[q] & 2) b[q] = g(lv->gx[q], lv->gy[q], lv->gz[q], par);
  free(fi);
}
static void set_bnd(const o3h* h, int l, int prob, const double* par, double* u, int zero_rest) {
  const o3lev* lv = &h->lv[l];
  const size_t N = (size_t)h->M * lv->S;
  o3fn f, g;
  pick(prob, &f, &g);
  for (size_t q = 0; q < N; ++q) {
    if (lv->flag[q] & 2) u[q] = g(lv->gx[q], lv->gy[q], lv->gz[q], par);
    else if (zero_rest) u[q] = 0.0;
  }
}

/* Level-0 operator on the macro-vertex values, assembled: row g adds, over
 * the group's members in slot order, their partial stencils (centre first,
 * then the directions inside the macro); coefficients of one column are added
 * in that order, the columns keep their first-appearance order; y_g is the
 * sequential sum over the row, written to every copy. */
static void apply0(const o3h* h, const double* x, double* y) {
  const o3lev* lv = &h->lv[0];
  const int n = lv->n, S = lv->S;
  for (int g = 0; g < lv->ng; ++g) {
    const int b = lv->gptr[g], e = lv->gptr[g + 1];
    int* col = malloc(sizeof(int) * 15 * (size_t)(e - b));
    double* val = malloc(sizeof(double) * 15 * (size_t)(e - b));
    int nc = 0;
    for (int q = b; q < e; ++q) {
      const int s = lv->mslot[q], i = lv->mi[q], j = lv->mj[q], k = lv->mk[q];
      const double* ps = lv->psK + 240 * (size_t)s + 15 * sig_of(n, i, j, k);
      for (int d = 0; d < 15; ++d) {
        const int a = i + DIR[d][0], bb = j + DIR[d][1], c = k + DIR[d][2];
        if (!inl(n, a, bb, c)) continue;
        const int gc = lv->gid[(size_t)s * S + lat3(n, a, bb, c)];
        int t = 0;
        while (t < nc && col[t] != gc) ++t;
        if (t == nc) { col[nc] = gc; val[nc] = ps[d]; ++nc; }
        else val[t] = val[t] + ps[d];
      }
    }
    double v = 0.0;
    for (int t = 0; t < nc; ++t) {
      const int gb = lv->gptr[col[t]];
      const double xv = x[(size_t)lv->mslot[gb] * S + lv->midx[gb]];
      v = t == 0 ? val[0] * xv : v + val[t] * xv;
    }
    for (int q = b; q < e; ++q) y[(size_t)lv->mslot[q] * S + lv->midx[q]] = v;
    free(col); free(val);
  }
}

/* level-0 CG (cg_level0 order, proj/src/multigrid.cpp:198-229) on the assembled operator */
int o3_cg0(const o3h* h, double* u, const double* b, double rel, double absf, int maxit, int* iters) {
  const o3lev* lv = &h->lv[0];
  const size_t N = (size_t)h->M * lv->S;
  double *r = malloc(8 * N), *p = malloc(8 * N), *ap = malloc(8 * N), *bz = malloc(8 * N);
  apply0(h, u, r);
  for (size_t q = 0; q < N; ++q) r[q] = (lv->flag[q] & 2) ? 0.0 : b[q] - r[q];
  memcpy(p, r, 8 * N);
  for (size_t q = 0; q < N; ++q) bz[q] = (lv->flag[q] & 2) ? 0.0 : b[q];
  double rr = o3_dot(h, 0, r, r);
  const double bn = sqrt(fmax(0.0, o3_dot(h, 0, bz, bz)));
  const double tol = rel * bn < absf ? absf : rel * bn;
  int it = 0, st = 0;
  while (sqrt(rr) > tol) {
    if (++it > maxit) { st = 1; break; }
    apply0(h, p, ap);
    for (size_t q = 0; q < N; ++q)
      if (lv->flag[q] & 2) ap[q] = 0.0;
    const double pap = o3_dot(h, 0, p, ap);
    if (pap <= 0.0) { st = 2; break; }
    const double alpha = rr / pap;
    for (size_t q = 0; q < N; ++q) {
      u[q] = u[q] + alpha * p[q];
      r[q] = r[q] + (-alpha) * ap[q];
    }
    const double rn = o3_dot(h, 0, r, r);
    const double beta = rn / rr;
    rr = rn;
    for (size_t q = 0; q < N; ++q) p[q] = p[q] * beta + r[q];
  }
  if (iters) *iters = it;
  free(r); free(p); free(ap); free(bz);
  return st;
}

static void vcycle(const o3h* h, int l, double* u, const double* b, int pre, int post, double rel, double absf,
                   int maxit) {
  if (l == 0) {
    o3_cg0(h, u, b, rel, absf, maxit, NULL);
    return;
  }
  const size_t Nf = (size_t)h->M * h->lv[l].S, Nc = (size_t)h->M * h->lv[l - 1].S;
  double *r = malloc(8 * Nf), *rc = malloc(8 * Nc), *ec = calloc(Nc, 8), *ef = malloc(8 * Nf);
  o3_gauss_seidel(h, l, u, b, pre);
  o3_residual(h, l, u, b, r);
  o3_restrict(h, l, r, rc);
  for (size_t q = 0; q < Nc; ++q)
    if (h->lv[l - 1].flag[q] & 2) rc[q] = 0.0;
  vcycle(h, l - 1, ec, rc, pre, post, rel, absf, maxit);
  o3_prolongate(h, l - 1, ec, ef);
  for (size_t q = 0; q < Nf; ++q) u[q] = u[q] + ef[q];
  o3_gauss_seidel(h, l, u, b, post);
  free(r); free(rc); free(ec); free(ef);
}

/* FMG (FinestPolicy::None); u[l], b[l] level arrays, w[l] = P u[l] on level l+1 */
int o3_fmg(const o3h* h, int prob, const double* par, int nu, int pre, int post, double rel, double absf, int maxit,
           double** u, double** b, double** w) {
  const int L = h->L;
  if (L < 1) return 3;
  for (int l = 0; l <= L; ++l) o3_rhs(h, l, prob, par, b[l]);
  set_bnd(h, 0, prob, par, u[0], 1);
  int st = o3_cg0(h, u[0], b[0], rel, absf, maxit, NULL);
  for (int l = 0; l < L; ++l) {
    o3_prolongate(h, l, u[l], w[l]);
    memcpy(u[l + 1], w[l], 8 * (size_t)h->M * h->lv[l + 1].S);
    set_bnd(h, l + 1, prob, par, u[l + 1], 0);
    for (int c = 0; c < nu; ++c) vcycle(h, l + 1, u[l + 1], b[l + 1], pre, post, rel, absf, maxit);
  }
  return st;
}

/* error_estimate (j = 1): e_base = u_L - w[L-1], e_coarser = u_L - P w[L-2];
 * per macro sums of e^T M_cell e (cells by base lattice index, then type) */
int o3_estimate(const o3h* h, const double* uL, double** w, double* out4, double* local_sums) {
  const int L = h->L;
  if (L < 2) return 1;
  const o3lev* lv = &h->lv[L];
  const int n = lv->n, S = lv->S;
  const size_t N = (size_t)h->M * S;
  double* pc = malloc(8 * N);
  o3_prolongate(h, L - 1, w[L - 2], pc);
  double gb = 0.0, gc = 0.0;
  for (int s = 0; s < h->M; ++s) {
    double qb = 0.0, qc = 0.0;
    for (int k = 0; k <= n; ++k)
      for (int j = 0; j <= n - k; ++j)
        for (int i = 0; i <= n - k - j; ++i)
          for (int ty = 0; ty < 6; ++ty) {
            int vi[4], ok = 1;
            for (int c = 0; c < 4 && ok; ++c) {
              int d[3];
              cvert(ty, c, d);
              ok = inl(n, i + d[0], j + d[1], k + d[2]);
              if (ok) vi[c] = lat3(n, i + d[0], j + d[1], k + d[2]);
            }
            if (!ok) continue;
            double eb[4], ec[4];
            for (int c = 0; c < 4; ++c) {
              const size_t o = (size_t)s * S + vi[c];
              eb[c] = uL[o] - w[L - 1][o];
              ec[c] = uL[o] - pc[o];
            }
            const double* Mt = lv->Mm + 96 * s + 16 * ty;
            for (int a = 0; a < 4; ++a) {
              const double rb = ((Mt[4 * a] * eb[0] + Mt[4 * a + 1] * eb[1]) + Mt[4 * a + 2] * eb[2]) + Mt[4 * a + 3] * eb[3];
              const double rc = ((Mt[4 * a] * ec[0] + Mt[4 * a + 1] * ec[1]) + Mt[4 * a + 2] * ec[2]) + Mt[4 * a + 3] * ec[3];
              qb = qb + eb[a] * rb;
              qc = qc + ec[a] * rc;
            }
          }
    local_sums[2 * s] = qb;
    local_sums[2 * s + 1] = qc;
    gb += qb;
    gc += qc;
  }
  free(pc);
  out4[0] = sqrt(fmax(0.0, gb));
  out4[1] = sqrt(fmax(0.0, gc));
  out4[2] = out4[1] > 0.0 ? out4[0] / out4[1] : 0.0;
  out4[3] = out4[2] * out4[0];
  return 0;
}

/* node coordinates of a level (owner coordinates for shared nodes), for tests */
void o3_coords(const o3h* h, int l, double* xyz_out) {
  const o3lev* lv = &h->lv[l];
  const size_t N = (size_t)h->M * lv->S;
  for (size_t q = 0; q < N; ++q) {
    xyz_out[3 * q] = lv->gx[q];
    xyz_out[3 * q + 1] = lv->gy[q];
    xyz_out[3 * q + 2] = lv->gz[q];
  }
}
