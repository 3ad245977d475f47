/*
 * gen.c -- multithreaded G1 "ideal-fusion patch fill" (SURVEY.md §8(d) generator rules,
 * DESIGN.md §3), the fast twin of scenes/fill.py:patch_fill for the large configs.
 *
 * INPUT PLUMBING shared by the CPU oracle and the CUDA path.  Like fill.py it holds none of
 * the rendering method's arithmetic (no membership ramp, combination weight, interpolation,
 * gradient, march or refinement): it writes clamped point-to-surface distances, the
 * direction factor <n, v^D> and a colour into the blocks that the angular
 * threshold (eq:angular_threshold) admits.
 *
 * Patch kinds (outward unit normal n(x) at voxel x, one-sided distance s(x), footprint):
 *   0 RECT  centre q, normal n, in-plane axes u, v, half extents hu, hv:
 *           s = <x - q, n>, footprint |<x-q,u>| <= hu and |<x-q,v>| <= hv   (== fill.py)
 *   1 DISK  centre q, normal n, radius hu:  s = <x - q, n>, footprint a^2 + b^2 <= hu^2
 *   2 CYL   lateral surface: axis through q along n, radius hu, half height hv:
 *           h = <x - q, n>, p = x - q - h n, s = |p| - hu, n(x) = p / |p|, footprint |h| <= hv
 * Rule (per direction D and voxel x): candidates are patches with <n(x), v^D> > cos(theta),
 * x inside the footprint and |s| <= tau + 2 s_vox; the smallest |s| wins (ties -> lower
 * patch id) and writes phi = clamp(s / tau, -1, 1), omega = <n(x), v^D>, rgb = colour.
 * Unwritten voxels hold phi = 1, omega = 0, rgb = 0.  A block (b, D) exists iff a voxel of it
 * was written.  Blocks come out sorted by (bx, by, bz, D) like fill.py.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -shared -fPIC -pthread (no fast-math, so the RECT
 * case reproduces fill.py's float64 arithmetic bit for bit).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { RECT = 0, DISK = 1, CYL = 2 };

typedef struct {
  int64_t b[3];
  int32_t D, p;
} triple;

typedef struct {
  int np;
  const int32_t *kind;
  const double *q, *n, *u, *v, *hu, *hv;
  const uint8_t *color;
  double s, tau, band, cos_t;
  triple *tri;
  int64_t ntri;
  int64_t *gstart; /* [ngroups + 1] */
  int64_t ngroups;
  uint8_t *keep;
  int64_t *outidx;
  int64_t nout;
} gen;

static const double VD[6][3] = {{1, 0, 0}, {-1, 0, 0}, {0, 1, 0}, {0, -1, 0}, {0, 0, 1}, {0, 0, -1}};

static int cmp_tri(const void *pa, const void *pb) {
  const triple *a = (const triple *)pa, *b = (const triple *)pb;
  for (int k = 0; k < 3; ++k)
    if (a->b[k] != b->b[k]) return a->b[k] < b->b[k] ? -1 : 1;
  if (a->D != b->D) return a->D < b->D ? -1 : 1;
  return (a->p > b->p) - (a->p < b->p);
}

static double dot3(const double *a, const double *b) {
  double r = a[0] * b[0] + a[1] * b[1];
  r += a[2] * b[2];
  return r;
}

/* candidate (block, D) triples of patch p */
static int emit(gen *g, int p, int64_t *cap) {
  const double bsz = 8.0 * g->s, band = g->band;
  const double *q = g->q + 3 * p, *n = g->n + 3 * p, *u = g->u + 3 * p, *v = g->v + 3 * p;
  const double hu = g->hu[p], hv = g->hv[p];
  const int kind = g->kind[p];
  double ext_u = hu, ext_v = hv, ext_n = band;
  if (kind == CYL) { ext_u = hu + band; ext_v = hu + band; ext_n = hv; }
  if (kind == DISK) { ext_v = hu; }
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int a = -1; a <= 1; a += 2)
    for (int b = -1; b <= 1; b += 2)
      for (int c = -1; c <= 1; c += 2)
        for (int k = 0; k < 3; ++k) {
          double x = q[k] + a * ext_u * u[k] + b * ext_v * v[k] + c * ext_n * n[k];
          if (x < lo[k]) lo[k] = x;
          if (x > hi[k]) hi[k] = x;
        }
  int64_t blo[3], bhi[3];
  for (int k = 0; k < 3; ++k) {
    blo[k] = (int64_t)floor(lo[k] / bsz - 1e-9);
    bhi[k] = (int64_t)floor(hi[k] / bsz + 1e-9);
  }
  int dmask = 0;
  for (int D = 0; D < 6; ++D) {
    double c = dot3(n, VD[D]);
    if (kind == CYL) c = sqrt(fmax(0.0, 1.0 - c * c)); /* best radial normal */
    if (c > g->cos_t) dmask |= 1 << D;
  }
  if (!dmask) return 0;
  const double rad = 0.5 * bsz * (fabs(n[0]) + fabs(n[1]) + fabs(n[2]));
  const double rfull = 0.5 * bsz * sqrt(3.0);
  for (int64_t bz = blo[2]; bz <= bhi[2]; ++bz)
    for (int64_t by = blo[1]; by <= bhi[1]; ++by)
      for (int64_t bx = blo[0]; bx <= bhi[0]; ++bx) {
        const double cen[3] = {(bx + 0.5) * bsz - q[0], (by + 0.5) * bsz - q[1], (bz + 0.5) * bsz - q[2]};
        if (kind == CYL) {
          const double h = dot3(cen, n);
          const double pr[3] = {cen[0] - h * n[0], cen[1] - h * n[1], cen[2] - h * n[2]};
          const double rho = sqrt(dot3(pr, pr));
          if (fabs(rho - hu) > band + rfull || fabs(h) > hv + rfull) continue;
        } else if (fabs(dot3(cen, n)) > band + rad) {
          continue;
        }
        for (int D = 0; D < 6; ++D) {
          if (!(dmask >> D & 1)) continue;
          if (g->ntri == *cap) {
            *cap = *cap ? 2 * *cap : 1 << 16;
            triple *t = (triple *)realloc(g->tri, sizeof(triple) * (size_t)*cap);
            if (!t) return -4;
            g->tri = t;
          }
          triple *t = &g->tri[g->ntri++];
          t->b[0] = bx; t->b[1] = by; t->b[2] = bz; t->D = D; t->p = p;
        }
      }
  return 0;
}

/* winner patch at voxel (i,j,k) of group G in direction D; returns 0 if unwritten */
static int voxel_eval(const gen *g, int64_t G, int64_t i, int64_t j, int64_t k, double *sp_out, double *om_out,
                      int *p_out) {
  const double x[3] = {(double)i * g->s, (double)j * g->s, (double)k * g->s};
  const int D = g->tri[g->gstart[G]].D;
  double best = INFINITY, bsp = 0, bom = 0;
  int bp = -1;
  for (int64_t t = g->gstart[G]; t < g->gstart[G + 1]; ++t) {
    const int p = g->tri[t].p;
    const double *q = g->q + 3 * p, *n = g->n + 3 * p;
    const double rel[3] = {x[0] - q[0], x[1] - q[1], x[2] - q[2]};
    double sp, om;
    if (g->kind[p] == CYL) {
      const double h = dot3(rel, n);
      if (fabs(h) > g->hv[p]) continue;
      const double pr[3] = {rel[0] - h * n[0], rel[1] - h * n[1], rel[2] - h * n[2]};
      const double rho = sqrt(dot3(pr, pr));
      if (!(rho > 0.0)) continue;
      sp = rho - g->hu[p];
      if (fabs(sp) > g->band) continue;
      om = dot3(pr, VD[D]) / rho;
      if (!(om > g->cos_t)) continue;
    } else {
      sp = dot3(rel, n);
      const double a = dot3(rel, g->u + 3 * p), b = dot3(rel, g->v + 3 * p);
      if (g->kind[p] == RECT) {
        if (!(fabs(a) <= g->hu[p] && fabs(b) <= g->hv[p])) continue;
      } else if (!(a * a + b * b <= g->hu[p] * g->hu[p])) {
        continue;
      }
      if (!(fabs(sp) <= g->band)) continue;
      om = dot3(n, VD[D]);
    }
    if (fabs(sp) < best) { best = fabs(sp); bsp = sp; bom = om; bp = p; }
  }
  if (bp < 0) return 0;
  *sp_out = bsp; *om_out = bom; *p_out = bp;
  return 1;
}

typedef struct {
  gen *g;
  int pass;
  int64_t next;
  int32_t *keys;
  float *sdf, *w;
  uint8_t *rgb;
} job;

static void *worker(void *arg) {
  job *J = (job *)arg;
  gen *g = J->g;
  for (;;) {
    const int64_t G0 = __atomic_fetch_add(&J->next, 64, __ATOMIC_RELAXED);
    if (G0 >= g->ngroups) break;
    const int64_t G1 = G0 + 64 < g->ngroups ? G0 + 64 : g->ngroups;
    for (int64_t G = G0; G < G1; ++G) {
      const triple *t0 = &g->tri[g->gstart[G]];
      if (J->pass == 1) {
        int any = 0;
        for (int l = 0; l < 512 && !any; ++l) {
          double sp, om;
          int p;
          any = voxel_eval(g, G, t0->b[0] * 8 + (l & 7), t0->b[1] * 8 + ((l >> 3) & 7), t0->b[2] * 8 + (l >> 6), &sp,
                           &om, &p);
        }
        g->keep[G] = (uint8_t)any;
      } else if (g->keep[G]) {
        const int64_t o = g->outidx[G];
        J->keys[4 * o + 0] = (int32_t)t0->b[0]; J->keys[4 * o + 1] = (int32_t)t0->b[1];
        J->keys[4 * o + 2] = (int32_t)t0->b[2]; J->keys[4 * o + 3] = t0->D;
        for (int l = 0; l < 512; ++l) {
          double sp, om;
          int p;
          float phi = 1.0f, w = 0.0f;
          uint8_t c[3] = {0, 0, 0};
          if (voxel_eval(g, G, t0->b[0] * 8 + (l & 7), t0->b[1] * 8 + ((l >> 3) & 7), t0->b[2] * 8 + (l >> 6), &sp, &om,
                         &p)) {
            double r = sp / g->tau;
            r = r < -1.0 ? -1.0 : (r > 1.0 ? 1.0 : r);
            phi = (float)r;
            w = (float)om;
            memcpy(c, g->color + 3 * p, 3);
          }
          J->sdf[512 * o + l] = phi;
          J->w[512 * o + l] = w;
          memcpy(J->rgb + 3 * (512 * o + l), c, 3);
        }
      }
    }
  }
  return NULL;
}

static void run(job *J, int nthreads) {
  J->next = 0;
  if (nthreads <= 1) { worker(J); return; }
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
  for (int i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, worker, J);
  for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
  free(th);
}

void scenegen_free(void *h) {
  gen *g = (gen *)h;
  if (!g) return;
  free(g->tri); free(g->gstart); free(g->keep); free(g->outidx);
  free(g);
}

/* Pass 1: candidate triples, grouping, which blocks exist.  Returns 0 or -4; *n_blocks = N. */
int scenegen_plan(int np, const int32_t *kind, const double *q, const double *n, const double *u, const double *v,
                  const double *hu, const double *hv, const uint8_t *color, double s, double tau, double theta,
                  int nthreads, void **out, int64_t *n_blocks) {
  gen *g = (gen *)calloc(1, sizeof(gen));
  if (!g) return -4;
  g->np = np; g->kind = kind; g->q = q; g->n = n; g->u = u; g->v = v; g->hu = hu; g->hv = hv; g->color = color;
  g->s = s; g->tau = tau; g->band = tau + 2.0 * s; g->cos_t = cos(theta);
  int64_t cap = 0;
  for (int p = 0; p < np; ++p)
    if (emit(g, p, &cap)) { scenegen_free(g); return -4; }
  qsort(g->tri, (size_t)g->ntri, sizeof(triple), cmp_tri);
  g->gstart = (int64_t *)malloc(sizeof(int64_t) * (size_t)(g->ntri + 1));
  if (!g->gstart) { scenegen_free(g); return -4; }
  for (int64_t t = 0; t < g->ntri; ++t)
    if (t == 0 || memcmp(g->tri[t].b, g->tri[t - 1].b, sizeof(g->tri[t].b)) || g->tri[t].D != g->tri[t - 1].D)
      g->gstart[g->ngroups++] = t;
  g->gstart[g->ngroups] = g->ntri;
  g->keep = (uint8_t *)calloc((size_t)g->ngroups + 1, 1);
  g->outidx = (int64_t *)malloc(sizeof(int64_t) * (size_t)(g->ngroups + 1));
  if (!g->keep || !g->outidx) { scenegen_free(g); return -4; }
  job J = {g, 1, 0, NULL, NULL, NULL, NULL};
  run(&J, nthreads);
  int64_t o = 0;
  for (int64_t G = 0; G < g->ngroups; ++G) {
    g->outidx[G] = o;
    o += g->keep[G];
  }
  g->nout = o;
  *n_blocks = o;
  *out = g;
  return 0;
}

/* Pass 2: write the N blocks into caller-owned arrays keys[N][4], sdf/weight[N][512], rgb[N][512][3]. */
void scenegen_fill(void *h, int nthreads, int32_t *keys, float *sdf, float *w, uint8_t *rgb) {
  job J = {(gen *)h, 2, 0, keys, sdf, w, rgb};
  run(&J, nthreads);
}
