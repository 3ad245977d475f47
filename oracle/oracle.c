/*
 * oracle.c -- plain, slow, fp64 CPU reference of the DTSDF raycast hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code, header,
 * table or constant with the CUDA path in paper_2301_12796_b200/ and never calls it.
 *
 * What it computes (readings R1-R31 in DESIGN.md §4):
 *   O1 ray          d~ = ((u-cx)/fx, (v-cy)/fy, 1), L = |d~|, r = R d~/L, o = t
 *                   (pinhole reprojection eq:reprojection)
 *   O2 lattice      t_k = k*Delta, k = ceil(zmin L/Delta) .. floor(zmax L/Delta)
 *                   ("probing the TSDF along the ray at regular intervals")
 *   O3 sample       per direction D: trilinear phi_D, omega_D over the 8 cell
 *                   corners; central-difference gradient n_D;
 *                   membership w_dir (eq:direction_weight, reading R1);
 *                   combination weight w_comb = w_dir(n_D) <n_D,-r> w_D
 *                   (eq:combine_weight) or, when no direction holding
 *                   data has a gradient, w_noGrad = w_D <v^D,-r> (eq:combine_tsdf_weight,
 *                   PAPER.md:265-270); f = sum W phi / sum W
 *   O4 crossing     first valid + -> valid - lattice pair
 *   O5 refinement   60 bisection steps in the bracket, or until it reaches the fp64
 *                   resolution of t (reading R5/R21)
 *   O6-O8           depth = camera z of the root; normal, colour, direction mask from the sample
 *                   at the final bracket end b (reading R32); zeros on a miss
 *
 * Brute force: every lattice point from zmin to zmax is evaluated; there is no range pass,
 * no block skipping and no hash -- the volume is a dense per-direction block-index grid.
 *
 * Pins: tests/test_oracle_*.py (closed forms, invariants, library reductions).
 * parity pinned: every exported function has at least one closed-form or reduction pin.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_BLOCK 8
#define OR_VPB 512

typedef struct {
  double s, tau, theta, delta;
  int64_t n;
  const int32_t *keys;  /* [n][4] (bx,by,bz,D) */
  const float *sdf;     /* [n][512] */
  const float *weight;  /* [n][512] */
  const uint8_t *rgb;   /* [n][512][3] or NULL */
  int64_t lo[3], dim[3];
  int32_t *grid;        /* [6][dim2][dim1][dim0] -> block id, -1 = unallocated */
  /* optional instrumentation: distinct records touched (algorithmic bytes) */
  uint8_t *touch_vox;   /* [n*512] sdf+weight record read by a sample evaluation */
  uint8_t *touch_rgb;   /* [n*512] colour record read by shading */
  uint8_t *touch_loc;   /* [dim2*dim1*dim0] block location whose presence was resolved */
} ovol;

/* v^D: X+, X-, Y+, Y-, Z+, Z- */
static const double VDIR[6][3] = {{1, 0, 0}, {-1, 0, 0}, {0, 1, 0}, {0, -1, 0}, {0, 0, 1}, {0, 0, -1}};

static int64_t floordiv8(int64_t i) { return (i >= 0) ? i / 8 : -((-i + 7) / 8); }

/* ---------------------------------------------------------------------------------------
 * volume: dense per-direction block grid.  Returns 0, -1 bad key, -2 duplicate key.
 * ------------------------------------------------------------------------------------- */
int oracle_volume_create(double s, double tau, double theta, double delta, int64_t n, const int32_t *keys,
                         const float *sdf, const float *weight, const uint8_t *rgb, void **out) {
  *out = NULL;
  ovol *v = (ovol *)calloc(1, sizeof(ovol));
  if (!v) return -4;
  v->s = s; v->tau = tau; v->theta = theta; v->delta = delta > 0 ? delta : s;
  v->n = n; v->keys = keys; v->sdf = sdf; v->weight = weight; v->rgb = rgb;
  int64_t lo[3] = {0, 0, 0}, hi[3] = {-1, -1, -1};
  for (int64_t b = 0; b < n; ++b) {
    if (keys[4 * b + 3] < 0 || keys[4 * b + 3] > 5) { free(v); return -1; }
    for (int a = 0; a < 3; ++a) {
      int64_t c = keys[4 * b + a];
      if (b == 0 || c < lo[a]) lo[a] = c;
      if (b == 0 || c > hi[a]) hi[a] = c;
    }
  }
  int64_t cells = 1;
  for (int a = 0; a < 3; ++a) {
    v->lo[a] = lo[a];
    v->dim[a] = n ? hi[a] - lo[a] + 1 : 0;
    cells *= v->dim[a];
  }
  v->grid = (int32_t *)malloc(sizeof(int32_t) * (size_t)(6 * (cells ? cells : 1)));
  if (!v->grid) { free(v); return -4; }
  for (int64_t i = 0; i < 6 * cells; ++i) v->grid[i] = -1;
  for (int64_t b = 0; b < n; ++b) {
    int64_t D = keys[4 * b + 3];
    int64_t gi = ((D * v->dim[2] + (keys[4 * b + 2] - lo[2])) * v->dim[1] + (keys[4 * b + 1] - lo[1])) * v->dim[0] +
                 (keys[4 * b + 0] - lo[0]);
    if (v->grid[gi] >= 0) { free(v->grid); free(v); return -2; }
    v->grid[gi] = (int32_t)b;
  }
  *out = v;
  return 0;
}

void oracle_volume_destroy(void *p) {
  ovol *v = (ovol *)p;
  if (!v) return;
  free(v->grid);
  free(v->touch_vox);
  free(v->touch_rgb);
  free(v->touch_loc);
  free(v);
}

/* enable instrumentation; returns 0 or -4 */
int oracle_enable_counting(void *p) {
  ovol *v = (ovol *)p;
  size_t cells = (size_t)(v->dim[0] * v->dim[1] * v->dim[2]);
  v->touch_vox = (uint8_t *)calloc((size_t)v->n * OR_VPB + 1, 1);
  v->touch_rgb = (uint8_t *)calloc((size_t)v->n * OR_VPB + 1, 1);
  v->touch_loc = (uint8_t *)calloc(cells + 1, 1);
  return (v->touch_vox && v->touch_rgb && v->touch_loc) ? 0 : -4;
}

/* counts[0] = distinct voxel records, [1] = distinct colour records, [2] = distinct locations */
void oracle_counts(void *p, int64_t *counts) {
  ovol *v = (ovol *)p;
  counts[0] = counts[1] = counts[2] = 0;
  if (!v->touch_vox) return;
  for (int64_t i = 0; i < v->n * OR_VPB; ++i) { counts[0] += v->touch_vox[i]; counts[1] += v->touch_rgb[i]; }
  for (int64_t i = 0; i < v->dim[0] * v->dim[1] * v->dim[2]; ++i) counts[2] += v->touch_loc[i];
}

/* block id holding voxel (i,j,k) of direction D, or -1 (unallocated / outside the grid) */
static int64_t block_of(const ovol *v, int D, int64_t i, int64_t j, int64_t k) {
  int64_t b[3] = {floordiv8(i) - v->lo[0], floordiv8(j) - v->lo[1], floordiv8(k) - v->lo[2]};
  for (int a = 0; a < 3; ++a)
    if (b[a] < 0 || b[a] >= v->dim[a]) return -1;
  int64_t cell = (b[2] * v->dim[1] + b[1]) * v->dim[0] + b[0];
  int32_t id = v->grid[(int64_t)D * v->dim[0] * v->dim[1] * v->dim[2] + cell];
  if (id >= 0 && v->touch_loc) __atomic_store_n(&v->touch_loc[cell], 1, __ATOMIC_RELAXED);
  return id;
}

/* record index of voxel (i,j,k) in direction D, or -1 */
static int64_t record_of(const ovol *v, int D, int64_t i, int64_t j, int64_t k) {
  int64_t b = block_of(v, D, i, j, k);
  if (b < 0) return -1;
  int64_t l = (i - 8 * floordiv8(i)) + 8 * (j - 8 * floordiv8(j)) + 64 * (k - 8 * floordiv8(k));
  return b * OR_VPB + l;
}

/* ---------------------------------------------------------------------------------------
 * O3(a): trilinear interpolation of cell (ci,cj,ck) with fractions fr.
 * Plain trilinear over the 8 corners including weight-0 voxels (reading R11); the direction
 * is absent (returns 0) unless all 8 corners lie in allocated blocks of D.
 * ------------------------------------------------------------------------------------- */
static int cell_interp(const ovol *v, int D, const int64_t c[3], const double fr[3], double *phi, double *omega,
                       int want_w, int64_t rec_out[8]) {
  double p = 0.0, w = 0.0;
  for (int q = 0; q < 8; ++q) {
    int dx = q & 1, dy = (q >> 1) & 1, dz = (q >> 2) & 1;
    int64_t r = record_of(v, D, c[0] + dx, c[1] + dy, c[2] + dz);
    if (r < 0) return 0;
    double wt = (dx ? fr[0] : 1.0 - fr[0]) * (dy ? fr[1] : 1.0 - fr[1]) * (dz ? fr[2] : 1.0 - fr[2]);
    p += wt * (double)v->sdf[r];
    if (want_w) w += wt * (double)v->weight[r];
    if (v->touch_vox) __atomic_store_n(&v->touch_vox[r], 1, __ATOMIC_RELAXED);
    if (rec_out) rec_out[q] = r;
  }
  *phi = p;
  if (want_w) *omega = w;
  return 1;
}

/* base cell and fractions of a world point (voxel (i,j,k) at (i,j,k)*s, reading R17) */
static void locate(const ovol *v, const double x[3], int64_t c[3], double fr[3]) {
  for (int a = 0; a < 3; ++a) {
    double g = x[a] / v->s;
    double fl = floor(g);
    c[a] = (int64_t)fl;
    fr[a] = g - fl;
  }
}

int oracle_trilinear(void *p, int D, const double x[3], double *phi, double *omega) {
  const ovol *v = (const ovol *)p;
  int64_t c[3];
  double fr[3];
  locate(v, x, c, fr);
  return cell_interp(v, D, c, fr, phi, omega, 1, NULL);
}

/* O3(c): g_a = (phi(cell + e_a) - phi(cell - e_a)) / (2s), the shifted cells taken with the
 * same fractions (central differences of trilinear phi at x +- s e_a, reading R7).
 * Returns 1 iff all six shifted cells are fully allocated in D. */
static int cell_gradient(const ovol *v, int D, const int64_t c[3], const double fr[3], double g[3]) {
  for (int a = 0; a < 3; ++a) {
    int64_t cp[3] = {c[0], c[1], c[2]}, cm[3] = {c[0], c[1], c[2]};
    cp[a] += 1;
    cm[a] -= 1;
    double pp, pm, dummy;
    if (!cell_interp(v, D, cp, fr, &pp, &dummy, 0, NULL)) return 0;
    if (!cell_interp(v, D, cm, fr, &pm, &dummy, 0, NULL)) return 0;
    g[a] = (pp - pm) / (2.0 * v->s);
  }
  return 1;
}

int oracle_gradient(void *p, int D, const double x[3], double g[3]) {
  const ovol *v = (const ovol *)p;
  int64_t c[3];
  double fr[3];
  locate(v, x, c, fr);
  return cell_gradient(v, D, c, fr, g);
}

/* eq:direction_weight with reading R1: clamp((theta - acos<n,v>) / (2 theta - pi/2), 0, 1) */
double oracle_w_dir(double cosang, double theta) {
  double c = cosang < -1.0 ? -1.0 : (cosang > 1.0 ? 1.0 : cosang);
  double w = (theta - acos(c)) / (2.0 * theta - M_PI / 2.0);
  return w < 0.0 ? 0.0 : (w > 1.0 ? 1.0 : w);
}

#define OR_EPS_GRAD 1e-3 /* reading R8: |g| <= 1e-3 m^-1 means "no gradient" */

typedef struct {
  int valid;
  double f, S;
  double W[6], nt[6][3], phi[6], omega[6];
  int present[6], data[6], has_grad[6];
  int regime; /* 1 = eq:combine_weight, 2 = eq:combine_tsdf_weight fallback */
  int64_t c[3];
  double fr[3];
} osample;

/* O3: F(x, r) */
static void eval_sample(const ovol *v, const double x[3], const double r[3], osample *o) {
  memset(o, 0, sizeof(*o));
  locate(v, x, o->c, o->fr);
  double sum_omega = 0.0;
  for (int D = 0; D < 6; ++D) {
    o->present[D] = cell_interp(v, D, o->c, o->fr, &o->phi[D], &o->omega[D], 1, NULL);
    if (o->present[D]) sum_omega += o->omega[D];
  }
  /* O3(b): W_D is proportional to omega_D in both regimes */
  if (!(sum_omega > 0.0)) return;
  double n[6][3];
  int any_grad = 0;
  for (int D = 0; D < 6; ++D) {
    o->data[D] = o->present[D] && o->omega[D] > 0.0; /* reading R8: "directions" = those holding data at x */
    if (!o->data[D]) continue;
    double g[3];
    if (cell_gradient(v, D, o->c, o->fr, g)) {
      double gn = sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
      if (gn > OR_EPS_GRAD) {
        o->has_grad[D] = 1;
        any_grad = 1;
        for (int a = 0; a < 3; ++a) n[D][a] = g[a] / gn;
      }
    }
  }
  double S = 0.0, F = 0.0;
  o->regime = any_grad ? 1 : 2;
  for (int D = 0; D < 6; ++D) {
    double W = 0.0;
    if (any_grad) {
      if (o->has_grad[D]) {
        double nv = n[D][0] * VDIR[D][0] + n[D][1] * VDIR[D][1] + n[D][2] * VDIR[D][2];
        double nr = -(n[D][0] * r[0] + n[D][1] * r[1] + n[D][2] * r[2]);
        W = oracle_w_dir(nv, v->theta) * (nr > 0.0 ? nr : 0.0) * o->omega[D]; /* eq:combine_weight */
        for (int a = 0; a < 3; ++a) o->nt[D][a] = n[D][a];
      }
    } else if (o->data[D]) {
      double vr = -(VDIR[D][0] * r[0] + VDIR[D][1] * r[1] + VDIR[D][2] * r[2]);
      W = o->omega[D] * (vr > 0.0 ? vr : 0.0); /* eq:combine_tsdf_weight */
      for (int a = 0; a < 3; ++a) o->nt[D][a] = VDIR[D][a];
    }
    o->W[D] = W;
    S += W;
    F += W * o->phi[D];
  }
  o->S = S;
  if (!(S > 0.0)) return; /* O3(e) */
  o->valid = 1;
  o->f = F / S;
}

/* exported single-sample evaluation for unit tests.
 * out[0]=valid out[1]=f out[2]=S out[3]=regime out[4..9]=W out[10..27]=nt out[28..33]=phi
 * out[34..39]=omega out[40..45]=present out[46..51]=has_grad */
int oracle_eval(void *p, const double x[3], const double r[3], double *out) {
  osample o;
  eval_sample((const ovol *)p, x, r, &o);
  out[0] = o.valid; out[1] = o.f; out[2] = o.S; out[3] = o.regime;
  for (int D = 0; D < 6; ++D) {
    out[4 + D] = o.W[D];
    for (int a = 0; a < 3; ++a) out[10 + 3 * D + a] = o.nt[D][a];
    out[28 + D] = o.phi[D];
    out[34 + D] = o.omega[D];
    out[40 + D] = o.present[D];
    out[46 + D] = o.has_grad[D];
  }
  return o.valid;
}

/* ---------------------------------------------------------------------------------------
 * O4-O8: one pixel
 * ------------------------------------------------------------------------------------- */
typedef struct {
  const ovol *v;
  double R[9], t[3];
  double fx, fy, cx, cy, zmin, zmax;
  int W, H;
  int64_t npix;
  const int32_t *uv; /* [npix][2] or NULL = all pixels row-major from row0 */
  int row0;
  double *depth, *normal;
  uint8_t *color, *mask;
  int32_t *nsamples; /* optional per-pixel lattice evaluations with a present direction */
  int64_t next;      /* work counter */
} ojob;

static void shade(const ovol *v, const osample *o, double *nrm, uint8_t *col, uint8_t *msk) {
  double N[3] = {0, 0, 0}, c[3] = {0, 0, 0};
  int m = 0;
  for (int D = 0; D < 6; ++D) {
    if (!(o->W[D] > 0.0)) continue;
    m |= 1 << D;
    for (int a = 0; a < 3; ++a) N[a] += o->W[D] * o->nt[D][a];
    if (v->rgb) {
      int64_t rec[8];
      double ph, om;
      cell_interp(v, D, o->c, o->fr, &ph, &om, 0, rec); /* corners are present (W_D > 0) */
      for (int q = 0; q < 8; ++q) {
        int dx = q & 1, dy = (q >> 1) & 1, dz = (q >> 2) & 1;
        double wt = (dx ? o->fr[0] : 1.0 - o->fr[0]) * (dy ? o->fr[1] : 1.0 - o->fr[1]) *
                    (dz ? o->fr[2] : 1.0 - o->fr[2]);
        for (int a = 0; a < 3; ++a) c[a] += o->W[D] * wt * (double)v->rgb[3 * rec[q] + a];
        if (v->touch_rgb) __atomic_store_n(&v->touch_rgb[rec[q]], 1, __ATOMIC_RELAXED);
      }
    }
  }
  double nn = sqrt(N[0] * N[0] + N[1] * N[1] + N[2] * N[2]);
  for (int a = 0; a < 3; ++a) nrm[a] = nn > 0.0 ? N[a] / nn : 0.0;
  for (int a = 0; a < 3; ++a) {
    double q = floor(c[a] / o->S + 0.5); /* reading R13: round half up, clamp at 255 */
    col[a] = (uint8_t)(q > 255.0 ? 255.0 : (q < 0.0 ? 0.0 : q));
  }
  *msk = (uint8_t)m;
}

static void render_pixel(ojob *J, int u, int vrow, int64_t out) {
  const ovol *v = J->v;
  double dt[3] = {(u - J->cx) / J->fx, (vrow - J->cy) / J->fy, 1.0};
  double L = sqrt(dt[0] * dt[0] + dt[1] * dt[1] + dt[2] * dt[2]);
  double r[3], o[3] = {J->t[0], J->t[1], J->t[2]};
  for (int a = 0; a < 3; ++a) r[a] = (J->R[3 * a] * dt[0] + J->R[3 * a + 1] * dt[1] + J->R[3 * a + 2] * dt[2]) / L;
  int64_t k0 = (int64_t)ceil(J->zmin * L / v->delta), k1 = (int64_t)floor(J->zmax * L / v->delta);
  int prev_valid = 0;
  double prev_f = 0.0;
  int32_t ns = 0;
  J->depth[out] = 0.0;
  for (int a = 0; a < 3; ++a) { J->normal[3 * out + a] = 0.0; J->color[3 * out + a] = 0; }
  J->mask[out] = 0;
  for (int64_t k = k0; k <= k1; ++k) {
    double t = (double)k * v->delta;
    double x[3] = {o[0] + t * r[0], o[1] + t * r[1], o[2] + t * r[2]};
    osample s;
    eval_sample(v, x, r, &s);
    for (int D = 0; D < 6; ++D) if (s.present[D]) { ns++; break; }
    if (s.valid && prev_valid && prev_f > 0.0 && s.f <= 0.0) {
      /* O5: bisection in [t_{k-1}, t_k]; invalid midpoints count as positive (R21) */
      double a = t - v->delta, b = t;
      for (int it = 0; it < 60; ++it) {
        double m = 0.5 * (a + b);
        if (!(m > a && m < b)) break; /* bracket at the fp64 resolution of t */
        double xm[3] = {o[0] + m * r[0], o[1] + m * r[1], o[2] + m * r[2]};
        osample sm;
        eval_sample(v, xm, r, &sm);
        if (!sm.valid || sm.f > 0.0) a = m; else b = m;
      }
      double ts = 0.5 * (a + b);
      J->depth[out] = ts / L; /* O6 */
      /* O7 (reading R32): shade at the final bracket end b -- a valid sample with f <= 0 at the
       * root to fp64 resolution, always on the surface side of a jump of F at the root */
      double xb[3] = {o[0] + b * r[0], o[1] + b * r[1], o[2] + b * r[2]};
      osample ss;
      eval_sample(v, xb, r, &ss);
      shade(v, &ss, &J->normal[3 * out], &J->color[3 * out], &J->mask[out]);
      break;
    }
    prev_valid = s.valid;
    prev_f = s.f;
  }
  if (J->nsamples) J->nsamples[out] = ns;
}

static void *worker(void *arg) {
  ojob *J = (ojob *)arg;
  const int64_t chunk = 64;
  for (;;) {
    int64_t i0 = __atomic_fetch_add(&J->next, chunk, __ATOMIC_RELAXED);
    if (i0 >= J->npix) break;
    int64_t i1 = i0 + chunk < J->npix ? i0 + chunk : J->npix;
    for (int64_t i = i0; i < i1; ++i) {
      int u, vr;
      if (J->uv) { u = J->uv[2 * i]; vr = J->uv[2 * i + 1]; }
      else { u = (int)(i % J->W); vr = J->row0 + (int)(i / J->W); }
      render_pixel(J, u, vr, i);
    }
  }
  return NULL;
}

/*
 * Render npix pixels of one view.  pose: world-from-camera 4x4 row-major; intr: fx fy cx cy
 * W H zmin zmax.  uv: [npix][2] pixel (column,row) list, or NULL for rows [row0, row0 + npix/W).
 * Outputs are indexed like the pixel list: depth [npix], normal [npix][3] (world, unit),
 * color [npix][3], mask [npix]; nsamples may be NULL.  nthreads <= 0 -> 1.
 */
void oracle_render(void *p, const double pose[16], const double intr[8], int64_t npix, const int32_t *uv, int row0,
                   int nthreads, double *depth, double *normal, uint8_t *color, uint8_t *mask, int32_t *nsamples) {
  ojob J;
  memset(&J, 0, sizeof(J));
  J.v = (const ovol *)p;
  for (int a = 0; a < 3; ++a) {
    for (int b = 0; b < 3; ++b) J.R[3 * a + b] = pose[4 * a + b];
    J.t[a] = pose[4 * a + 3];
  }
  J.fx = intr[0]; J.fy = intr[1]; J.cx = intr[2]; J.cy = intr[3];
  J.W = (int)intr[4]; J.H = (int)intr[5]; J.zmin = intr[6]; J.zmax = intr[7];
  J.npix = npix; J.uv = uv; J.row0 = row0;
  J.depth = depth; J.normal = normal; J.color = color; J.mask = mask; J.nsamples = nsamples;
  if (nthreads <= 1) { worker(&J); return; }
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
  for (int i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, worker, &J);
  for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
  free(th);
}

/* =======================================================================================
 * NEXT-1: the view-dependent combined TSDF (Lemma 1, PAPER.md:182-186;
 * PAPER.md:251-263; implementation note PAPER.md:610) and its raycast.  Readings R33-R40 of
 * DESIGN.md §4.  Everything is a pure function of (volume, source camera): a combined voxel is
 * evaluated on demand from the directional voxels, nothing is cached.
 * ===================================================================================== */
typedef struct {
  double R[9], t[3];
  double fx, fy, cx, cy, zmin, zmax;
  int W, H;
  double margin; /* fraction of the image size added on every side (1/8) */
  int mode;      /* 0: eq:combine_weight / eq:combine_tsdf_weight (R34); 1: Algorithm 1 (R53-R57) */
  double w_floor;/* Algorithm 1: directions need a stored weight above this (R53) */
  const ovol *vprev; /* R58: the volume the combined TSDF was computed from, when fusion has changed the
                      * volume since (NULL: combined from the current volume) */
} ocam;

static void cam_from(ocam *c, const double pose[16], const double intr[8], double margin) {
  for (int a = 0; a < 3; ++a) {
    for (int b = 0; b < 3; ++b) c->R[3 * a + b] = pose[4 * a + b];
    c->t[a] = pose[4 * a + 3];
  }
  c->fx = intr[0]; c->fy = intr[1]; c->cx = intr[2]; c->cy = intr[3];
  c->W = (int)intr[4]; c->H = (int)intr[5]; c->zmin = intr[6]; c->zmax = intr[7];
  c->margin = margin;
  c->mode = 0;
  c->w_floor = 0.0;
  c->vprev = NULL;
}

/* R33: voxel (i,j,k) lies in the source view frustum widened by margin*W / margin*H pixels on
 * every side ("selecting voxels slightly beyond the camera frustum (±1/8 image size)",
 * PAPER.md:262) and inside [zmin, zmax] in camera z.  Evaluated left to right, one rounding per
 * operation (the CUDA path evaluates the same expression with the same roundings). */
static int in_frustum(const ocam *c, double s, int64_t i, int64_t j, int64_t k) {
  double x[3] = {(double)i * s, (double)j * s, (double)k * s};
  double d[3] = {x[0] - c->t[0], x[1] - c->t[1], x[2] - c->t[2]};
  double xc[3];
  for (int a = 0; a < 3; ++a) xc[a] = c->R[a] * d[0] + c->R[3 + a] * d[1] + c->R[6 + a] * d[2];
  if (!(xc[2] >= c->zmin && xc[2] <= c->zmax)) return 0;
  double u = c->fx * xc[0] / xc[2] + c->cx, v = c->fy * xc[1] / xc[2] + c->cy;
  double mu = c->margin * (double)c->W, mv = c->margin * (double)c->H;
  return u >= -mu && u <= (double)(c->W - 1) + mu && v >= -mv && v <= (double)(c->H - 1) + mv;
}

typedef struct {
  int valid;    /* S > 0 */
  double sdf;   /* sum W phi / S */
  double S;     /* sum W: the combined voxel's weight */
  double rgb[3];/* sum W c_D / S (reals) */
  int mask;     /* bit D: W_D > 0 */
} ocvox;

/* R34: the combined value of the voxel at integer position (i,j,k) ("calculating the combined
 * SDF for every voxel in the view frustum") with the combination weights of
 * eq:combine_weight / eq:combine_tsdf_weight; the gradient
 * n^D from "the SDF values stored in the 6 neighboring voxels", i.e. central
 * differences (phi(i+e_a) - phi(i-e_a)) / 2s; r = the normalised ray from the source camera
 * centre to the voxel.  Directions, gradient presence and the regime choice as O3 (R8-R10). */
static void combine_voxel_alg1(const ovol *v, const ocam *c, int64_t i, int64_t j, int64_t k, ocvox *o);

static void combine_voxel(const ovol *v, const ocam *c, int64_t i, int64_t j, int64_t k, ocvox *o) {
  if (c->mode == 1) { combine_voxel_alg1(v, c, i, j, k, o); return; }
  memset(o, 0, sizeof(*o));
  if (!in_frustum(c, v->s, i, j, k)) return;
  double x[3] = {(double)i * v->s, (double)j * v->s, (double)k * v->s};
  double r[3] = {x[0] - c->t[0], x[1] - c->t[1], x[2] - c->t[2]};
  double rl = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
  if (!(rl > 0.0)) return;
  for (int a = 0; a < 3; ++a) r[a] /= rl;
  const int64_t vi[3] = {i, j, k};
  double phi[6], om[6], n[6][3];
  int64_t rec[6];
  int data[6], hg[6], any_grad = 0;
  for (int D = 0; D < 6; ++D) {
    data[D] = hg[D] = 0;
    rec[D] = record_of(v, D, i, j, k);
    if (rec[D] < 0) continue;
    phi[D] = (double)v->sdf[rec[D]];
    om[D] = (double)v->weight[rec[D]];
    data[D] = om[D] > 0.0;
    if (!data[D]) continue;
    double g[3];
    int ok = 1;
    for (int a = 0; a < 3 && ok; ++a) {
      int64_t p[3] = {vi[0], vi[1], vi[2]}, m[3] = {vi[0], vi[1], vi[2]};
      p[a] += 1;
      m[a] -= 1;
      int64_t rp = record_of(v, D, p[0], p[1], p[2]), rm = record_of(v, D, m[0], m[1], m[2]);
      if (rp < 0 || rm < 0) { ok = 0; break; }
      g[a] = ((double)v->sdf[rp] - (double)v->sdf[rm]) / (2.0 * v->s);
    }
    if (!ok) continue;
    double gn = sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
    if (gn > OR_EPS_GRAD) {
      hg[D] = 1;
      any_grad = 1;
      for (int a = 0; a < 3; ++a) n[D][a] = g[a] / gn;
    }
  }
  double S = 0.0, F = 0.0, C[3] = {0, 0, 0};
  int m = 0;
  for (int D = 0; D < 6; ++D) {
    double W = 0.0;
    if (any_grad) {
      if (hg[D]) {
        double nv = n[D][0] * VDIR[D][0] + n[D][1] * VDIR[D][1] + n[D][2] * VDIR[D][2];
        double nr = -(n[D][0] * r[0] + n[D][1] * r[1] + n[D][2] * r[2]);
        W = oracle_w_dir(nv, v->theta) * (nr > 0.0 ? nr : 0.0) * om[D]; /* eq:combine_weight */
      }
    } else if (data[D]) {
      double vr = -(VDIR[D][0] * r[0] + VDIR[D][1] * r[1] + VDIR[D][2] * r[2]);
      W = om[D] * (vr > 0.0 ? vr : 0.0); /* eq:combine_tsdf_weight */
    }
    if (!(W > 0.0)) continue;
    m |= 1 << D;
    S += W;
    F += W * phi[D];
    if (v->rgb)
      for (int a = 0; a < 3; ++a) C[a] += W * (double)v->rgb[3 * rec[D] + a];
  }
  if (!(S > 0.0)) return;
  o->valid = 1;
  o->S = S;
  o->sdf = F / S;
  for (int a = 0; a < 3; ++a) o->rgb[a] = C[a] / S;
  o->mask = m;
}


/* ---------------------------------------------------------------------------------------
 * NEXT-4: Algorithm 1 "Compute Combined TSDF" (prose P:217-226) at an integer
 * voxel position, readings R53-R57:
 *   R53 a direction D takes part iff allocated at the voxel, its stored weight exceeds w_floor
 *       (0 by default: ">0"), its 6-neighbour gradient exists (|g| > 1e-3) and is valid w.r.t.
 *       the direction vector, w_dir(<n^D, v^D>) > 0 ("ignoring information from points with
 *       invalid gradients")
 *   R54 F = taking-part directions with phi_D(p) > 0 (free), O = those with phi_D(p) <= 0
 *   R55 for D in F: q = first zero transition of Phi^D from p towards the camera (-r): samples
 *       p - k s r, k = 1 .. floor(|p - c| / s), the march ends without a transition (q = none) at
 *       the first sample where D is absent; bisection in the bracket (invalid midpoints positive)
 *   R56 D's free space stands iff q = none or no other direction D~ has Phi^D~(q) < 0 (as
 *       printed) with a gradient n^D~(q) (central differences, R7) and <n^D~(q), -r> > 0;
 *       freespace = OR over F.  (A direction storing the same surface as D is ~0 at D's own root,
 *       so its sign there is decided by rounding: such voxels may differ between implementations
 *       and count against the parity budget, reading R22.)
 *   R57 freespace -> the stored-weight average of the F directions; else of the O directions;
 *       else invalid ("all congruent directions are combined as weighted sum using the fused voxel
 *       weights")
 * ------------------------------------------------------------------------------------- */
static int dir_value(const ovol *v, int D, const double x[3], double *phi) {
  int64_t cc[3];
  double fr[3], om;
  locate(v, x, cc, fr);
  return cell_interp(v, D, cc, fr, phi, &om, 0, NULL);
}

static int dir_normal(const ovol *v, int D, const double x[3], double n[3]) {
  int64_t cc[3];
  double fr[3], g[3];
  locate(v, x, cc, fr);
  if (!cell_gradient(v, D, cc, fr, g)) return 0;
  double gn = sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
  if (!(gn > OR_EPS_GRAD)) return 0;
  for (int a = 0; a < 3; ++a) n[a] = g[a] / gn;
  return 1;
}

static void combine_voxel_alg1(const ovol *v, const ocam *c, int64_t i, int64_t j, int64_t k, ocvox *o) {
  memset(o, 0, sizeof(*o));
  if (!in_frustum(c, v->s, i, j, k)) return;
  double x[3] = {(double)i * v->s, (double)j * v->s, (double)k * v->s};
  double r[3] = {x[0] - c->t[0], x[1] - c->t[1], x[2] - c->t[2]};
  double dist = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
  if (!(dist > 0.0)) return;
  for (int a = 0; a < 3; ++a) r[a] /= dist;
  const int64_t vi[3] = {i, j, k};
  double phi[6], om[6];
  int64_t rec[6];
  int part[6];
  for (int D = 0; D < 6; ++D) {
    part[D] = 0;
    rec[D] = record_of(v, D, i, j, k);
    if (rec[D] < 0) continue;
    phi[D] = (double)v->sdf[rec[D]];
    om[D] = (double)v->weight[rec[D]];
    if (!(om[D] > c->w_floor)) continue;
    double g[3];
    int ok = 1;
    for (int a = 0; a < 3 && ok; ++a) {
      int64_t pp[3] = {vi[0], vi[1], vi[2]}, mm[3] = {vi[0], vi[1], vi[2]};
      pp[a] += 1;
      mm[a] -= 1;
      int64_t rp = record_of(v, D, pp[0], pp[1], pp[2]), rm = record_of(v, D, mm[0], mm[1], mm[2]);
      if (rp < 0 || rm < 0) { ok = 0; break; }
      g[a] = ((double)v->sdf[rp] - (double)v->sdf[rm]) / (2.0 * v->s);
    }
    if (!ok) continue;
    double gn = sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
    if (!(gn > OR_EPS_GRAD)) continue;
    double nv = (g[0] * VDIR[D][0] + g[1] * VDIR[D][1] + g[2] * VDIR[D][2]) / gn;
    if (!(oracle_w_dir(nv, v->theta) > 0.0)) continue;
    part[D] = 1;
  }
  int freespace = 0, any_free = 0, any_occ = 0;
  const int64_t K = (int64_t)floor(dist / v->s);
  for (int D = 0; D < 6; ++D) {
    if (!part[D]) continue;
    if (!(phi[D] > 0.0)) { any_occ = 1; continue; }
    any_free = 1;
    if (freespace) continue;
    /* R55: back-march towards the camera in Phi^D */
    double prev_t = 0.0, qt = -1.0;
    for (int64_t kk = 1; kk <= K; ++kk) {
      double t = (double)kk * v->s, y[3] = {x[0] - t * r[0], x[1] - t * r[1], x[2] - t * r[2]}, f;
      if (!dir_value(v, D, y, &f)) break; /* D absent: no transition observed */
      if (f <= 0.0) {
        double a = prev_t, b = t;
        for (int it = 0; it < 50; ++it) {
          double m = 0.5 * (a + b), ym[3] = {x[0] - m * r[0], x[1] - m * r[1], x[2] - m * r[2]}, fm;
          if (!(m > a && m < b)) break;
          if (!dir_value(v, D, ym, &fm) || fm > 0.0) a = m; else b = m;
        }
        qt = 0.5 * (a + b);
        break;
      }
      prev_t = t;
    }
    if (qt < 0.0) { freespace = 1; continue; }
    double q[3] = {x[0] - qt * r[0], x[1] - qt * r[1], x[2] - qt * r[2]};
    int conflict = 0;
    for (int E = 0; E < 6 && !conflict; ++E) {
      if (E == D) continue;
      double fe, ne[3];
      if (!dir_value(v, E, q, &fe) || !(fe < 0.0)) continue; /* P:204 "Phi^D~(q) < 0" */
      if (!dir_normal(v, E, q, ne)) continue;
      if (-(ne[0] * r[0] + ne[1] * r[1] + ne[2] * r[2]) > 0.0) conflict = 1;
    }
    if (!conflict) freespace = 1;
  }
  if (!any_free && !any_occ) return;
  const int use_free = freespace;
  if (!use_free && !any_occ) return;
  double S = 0.0, F = 0.0, C[3] = {0, 0, 0};
  int m = 0;
  for (int D = 0; D < 6; ++D) {
    if (!part[D] || ((phi[D] > 0.0) != (use_free != 0))) continue;
    S += om[D];
    F += om[D] * phi[D];
    if (v->rgb)
      for (int a = 0; a < 3; ++a) C[a] += om[D] * (double)v->rgb[3 * rec[D] + a];
    m |= 1 << D;
  }
  if (!(S > 0.0)) return;
  o->valid = 1;
  o->S = S;
  o->sdf = F / S;
  for (int a = 0; a < 3; ++a) o->rgb[a] = C[a] / S;
  o->mask = m;
}

/* a voxel "has data" iff some direction's block holding it is allocated with stored weight > 0 */
static int has_data(const ovol *v, int64_t i, int64_t j, int64_t k) {
  for (int D = 0; D < 6; ++D) {
    int64_t r = record_of(v, D, i, j, k);
    if (r >= 0 && v->weight[r] > 0.0f) return 1;
  }
  return 0;
}

/* R58: "Voxels that receive data for the first time are always directly added to the combined
 * TSDF".  After fusion changed the volume from c->vprev (the volume the combined TSDF
 * was computed from) to v, a voxel that had no data in vprev and has data in v takes its combined
 * value from v; every other voxel keeps the value combined from vprev (stale until the next
 * recombination, eqs. condition_1-4).  Without vprev: the combined value from v. */
static void combined_at(const ovol *v, const ocam *c, int64_t i, int64_t j, int64_t k, ocvox *o) {
  if (c->vprev) {
    const int first = !has_data(c->vprev, i, j, k) && has_data(v, i, j, k);
    combine_voxel(first ? v : c->vprev, c, i, j, k, o);
    return;
  }
  combine_voxel(v, c, i, j, k, o);
}

/* R35: the stored colour of a combined voxel is the u8 value min(255, floor(c + 1/2)) */
static uint8_t u8_round(double c) {
  double q = floor(c + 0.5);
  return (uint8_t)(q > 255.0 ? 255.0 : (q < 0.0 ? 0.0 : q));
}

/* Combined voxels of a list of integer positions (element-wise parity / pins).
 * ijk [n][3]; outputs valid[n], sdf[n], S[n], rgb[n][3] (u8 after R35), mask[n]. */
static void combined_voxels(const ovol *v, const ovol *vprev, const double pose[16], const double intr[8],
                            double margin, int mode, double w_floor, int64_t n, const int64_t *ijk, int32_t *valid,
                            double *sdf, double *S, uint8_t *rgb, uint8_t *mask) {
  ocam c;
  cam_from(&c, pose, intr, margin);
  c.mode = mode;
  c.w_floor = w_floor;
  c.vprev = vprev;
  for (int64_t q = 0; q < n; ++q) {
    ocvox o;
    combined_at(v, &c, ijk[3 * q], ijk[3 * q + 1], ijk[3 * q + 2], &o);
    valid[q] = o.valid;
    sdf[q] = o.valid ? o.sdf : 0.0;
    S[q] = o.S;
    for (int a = 0; a < 3; ++a) rgb[3 * q + a] = o.valid ? u8_round(o.rgb[a]) : 0;
    mask[q] = (uint8_t)o.mask;
  }
}

void oracle_combined_voxels_mode(void *p, const double pose[16], const double intr[8], double margin, int mode,
                                 double w_floor, int64_t n, const int64_t *ijk, int32_t *valid, double *sdf, double *S,
                                 uint8_t *rgb, uint8_t *mask) {
  combined_voxels((const ovol *)p, NULL, pose, intr, margin, mode, w_floor, n, ijk, valid, sdf, S, rgb, mask);
}

/* R58: combined voxels after fusion changed the volume `before` (the one combined) to `after` */
void oracle_combined_voxels_update(void *before, void *after, const double pose[16], const double intr[8],
                                   double margin, int mode, double w_floor, int64_t n, const int64_t *ijk,
                                   int32_t *valid, double *sdf, double *S, uint8_t *rgb, uint8_t *mask) {
  combined_voxels((const ovol *)after, (const ovol *)before, pose, intr, margin, mode, w_floor, n, ijk, valid, sdf,
                  S, rgb, mask);
}

/* R36: the combined field is a regular TSDF ("can then be used like a regular
 * TSDF"): plain trilinear of the combined sdf over the 8 cell corners, valid iff all 8 corners
 * are valid combined voxels. */
static int ccell(const ovol *v, const ocam *c, const int64_t cc[3], const double fr[3], double *phi, ocvox corner[8]) {
  double ph = 0.0;
  for (int q = 0; q < 8; ++q) {
    int dx = q & 1, dy = (q >> 1) & 1, dz = (q >> 2) & 1;
    ocvox o;
    combined_at(v, c, cc[0] + dx, cc[1] + dy, cc[2] + dz, &o);
    if (!o.valid) return 0;
    double wt = (dx ? fr[0] : 1.0 - fr[0]) * (dy ? fr[1] : 1.0 - fr[1]) * (dz ? fr[2] : 1.0 - fr[2]);
    ph += wt * o.sdf;
    if (corner) corner[q] = o;
  }
  *phi = ph;
  return 1;
}

/* R37: shading of a combined-TSDF hit at the bracket end b (as R32):
 *   normal = normalised central-difference gradient of the trilinear combined field at +-s
 *            (R7 on the combined field) when the six shifted cells are valid and |g| > 1e-3;
 *            otherwise the gradient of the cell's own trilinear interpolant when |g| > 1e-3;
 *            otherwise 0;
 *   colour = min(255, floor(trilinear of the corners' u8 colours + 1/2));
 *   mask   = OR of the direction masks of the corners whose trilinear weight is >= 1/8 (at least
 *            one corner qualifies, so a hit has a nonempty mask; a plain OR over all 8 corners
 *            would depend on which side of a voxel plane a root lying on that plane -- e.g. a
 *            floor at z = 0 -- is refined to). */
static void cshade(const ovol *v, const ocam *c, const int64_t cc[3], const double fr[3], double *nrm, uint8_t *col,
                   uint8_t *msk) {
  ocvox cor[8];
  double ph;
  nrm[0] = nrm[1] = nrm[2] = 0.0;
  col[0] = col[1] = col[2] = 0;
  *msk = 0;
  if (!ccell(v, c, cc, fr, &ph, cor)) return;
  double g[3];
  int ok = 1;
  for (int a = 0; a < 3 && ok; ++a) {
    int64_t cp[3] = {cc[0], cc[1], cc[2]}, cm[3] = {cc[0], cc[1], cc[2]};
    cp[a] += 1;
    cm[a] -= 1;
    double pp, pm;
    if (!ccell(v, c, cp, fr, &pp, NULL) || !ccell(v, c, cm, fr, &pm, NULL)) { ok = 0; break; }
    g[a] = (pp - pm) / (2.0 * v->s);
  }
  double gn = ok ? sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]) : 0.0;
  if (!(gn > OR_EPS_GRAD)) {
    /* d/dx_a of sum_q wt_q(fr) phi_q, with d fr_a / d x_a = 1/s */
    for (int a = 0; a < 3; ++a) {
      double acc = 0.0;
      for (int q = 0; q < 8; ++q) {
        int bit[3] = {q & 1, (q >> 1) & 1, (q >> 2) & 1};
        double wt = 1.0;
        for (int e = 0; e < 3; ++e) {
          if (e == a) wt *= bit[e] ? 1.0 : -1.0;
          else wt *= bit[e] ? fr[e] : 1.0 - fr[e];
        }
        acc += wt * cor[q].sdf;
      }
      g[a] = acc / v->s;
    }
    gn = sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
  }
  if (gn > OR_EPS_GRAD)
    for (int a = 0; a < 3; ++a) nrm[a] = g[a] / gn;
  double cs[3] = {0, 0, 0};
  int m = 0;
  for (int q = 0; q < 8; ++q) {
    int dx = q & 1, dy = (q >> 1) & 1, dz = (q >> 2) & 1;
    double wt = (dx ? fr[0] : 1.0 - fr[0]) * (dy ? fr[1] : 1.0 - fr[1]) * (dz ? fr[2] : 1.0 - fr[2]);
    for (int a = 0; a < 3; ++a) cs[a] += wt * (double)u8_round(cor[q].rgb[a]);
    if (wt >= 0.125) m |= cor[q].mask;
  }
  for (int a = 0; a < 3; ++a) col[a] = u8_round(cs[a]);
  *msk = (uint8_t)m;
}

typedef struct {
  const ovol *v;
  ocam src;          /* camera the combined TSDF was computed for */
  ojob J;            /* rendering camera, pixels and outputs */
} ocjob;

/* O1-O6 on the combined field (same lattice, crossing rule and bisection as the direct path,
 * PAPER.md:178), R37 shading */
static void render_pixel_combined(ocjob *C, int u, int vrow, int64_t out) {
  ojob *J = &C->J;
  const ovol *v = C->v;
  double dt[3] = {(u - J->cx) / J->fx, (vrow - J->cy) / J->fy, 1.0};
  double L = sqrt(dt[0] * dt[0] + dt[1] * dt[1] + dt[2] * dt[2]);
  double r[3], o[3] = {J->t[0], J->t[1], J->t[2]};
  for (int a = 0; a < 3; ++a) r[a] = (J->R[3 * a] * dt[0] + J->R[3 * a + 1] * dt[1] + J->R[3 * a + 2] * dt[2]) / L;
  int64_t k0 = (int64_t)ceil(J->zmin * L / v->delta), k1 = (int64_t)floor(J->zmax * L / v->delta);
  int prev_valid = 0;
  double prev_f = 0.0;
  J->depth[out] = 0.0;
  for (int a = 0; a < 3; ++a) { J->normal[3 * out + a] = 0.0; J->color[3 * out + a] = 0; }
  J->mask[out] = 0;
  for (int64_t k = k0; k <= k1; ++k) {
    double t = (double)k * v->delta;
    double x[3] = {o[0] + t * r[0], o[1] + t * r[1], o[2] + t * r[2]};
    int64_t cc[3];
    double fr[3], f = 0.0;
    locate(v, x, cc, fr);
    int valid = ccell(v, &C->src, cc, fr, &f, NULL);
    if (valid && prev_valid && prev_f > 0.0 && f <= 0.0) {
      double a = t - v->delta, b = t;
      for (int it = 0; it < 60; ++it) {
        double m = 0.5 * (a + b);
        if (!(m > a && m < b)) break;
        double xm[3] = {o[0] + m * r[0], o[1] + m * r[1], o[2] + m * r[2]};
        int64_t cm[3];
        double fm[3], ff = 0.0;
        locate(v, xm, cm, fm);
        int vm = ccell(v, &C->src, cm, fm, &ff, NULL);
        if (!vm || ff > 0.0) a = m; else b = m;
      }
      J->depth[out] = 0.5 * (a + b) / L;
      double xb[3] = {o[0] + b * r[0], o[1] + b * r[1], o[2] + b * r[2]};
      int64_t cb[3];
      double fb[3];
      locate(v, xb, cb, fb);
      cshade(v, &C->src, cb, fb, &J->normal[3 * out], &J->color[3 * out], &J->mask[out]);
      break;
    }
    prev_valid = valid;
    prev_f = f;
  }
}

static void *worker_combined(void *arg) {
  ocjob *C = (ocjob *)arg;
  ojob *J = &C->J;
  const int64_t chunk = 16;
  for (;;) {
    int64_t i0 = __atomic_fetch_add(&J->next, chunk, __ATOMIC_RELAXED);
    if (i0 >= J->npix) break;
    int64_t i1 = i0 + chunk < J->npix ? i0 + chunk : J->npix;
    for (int64_t i = i0; i < i1; ++i) {
      int u, vr;
      if (J->uv) { u = J->uv[2 * i]; vr = J->uv[2 * i + 1]; }
      else { u = (int)(i % J->W); vr = J->row0 + (int)(i / J->W); }
      render_pixel_combined(C, u, vr, i);
    }
  }
  return NULL;
}

/* Render npix pixels of the view (pose, intr) from the combined TSDF of the source camera
 * (src_pose, src_intr, margin).  Argument conventions as oracle_render. */
static void render_combined(const ovol *v, const ovol *vprev, const double src_pose[16], const double src_intr[8],
                            double margin, int mode, double w_floor, const double pose[16], const double intr[8],
                            int64_t npix, const int32_t *uv, int row0, int nthreads, double *depth, double *normal,
                            uint8_t *color, uint8_t *mask) {
  ocjob C;
  memset(&C, 0, sizeof(C));
  C.v = v;
  cam_from(&C.src, src_pose, src_intr, margin);
  C.src.mode = mode;
  C.src.w_floor = w_floor;
  C.src.vprev = vprev;
  ojob *J = &C.J;
  J->v = C.v;
  for (int a = 0; a < 3; ++a) {
    for (int b = 0; b < 3; ++b) J->R[3 * a + b] = pose[4 * a + b];
    J->t[a] = pose[4 * a + 3];
  }
  J->fx = intr[0]; J->fy = intr[1]; J->cx = intr[2]; J->cy = intr[3];
  J->W = (int)intr[4]; J->H = (int)intr[5]; J->zmin = intr[6]; J->zmax = intr[7];
  J->npix = npix; J->uv = uv; J->row0 = row0;
  J->depth = depth; J->normal = normal; J->color = color; J->mask = mask;
  if (nthreads <= 1) { worker_combined(&C); return; }
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
  for (int i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, worker_combined, &C);
  for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
  free(th);
}

void oracle_render_combined_mode(void *p, const double src_pose[16], const double src_intr[8], double margin,
                                 int mode, double w_floor, const double pose[16], const double intr[8], int64_t npix,
                                 const int32_t *uv, int row0, int nthreads, double *depth, double *normal,
                                 uint8_t *color, uint8_t *mask) {
  render_combined((const ovol *)p, NULL, src_pose, src_intr, margin, mode, w_floor, pose, intr, npix, uv, row0,
                  nthreads, depth, normal, color, mask);
}

/* R58: render the combined TSDF after fusion changed the volume `before` (the one combined) to `after` */
void oracle_render_combined_update(void *before, void *after, const double src_pose[16], const double src_intr[8],
                                   double margin, int mode, double w_floor, const double pose[16], const double intr[8],
                                   int64_t npix, const int32_t *uv, int row0, int nthreads, double *depth,
                                   double *normal, uint8_t *color, uint8_t *mask) {
  render_combined((const ovol *)after, (const ovol *)before, src_pose, src_intr, margin, mode, w_floor, pose, intr,
                  npix, uv, row0, nthreads, depth, normal, color, mask);
}

/* Conditional combination (eqs. condition_1-4): recombine iff
 *   framesSinceStart < boot  OR  framesSinceLastUpdate > stale  OR
 *   ||t - t_last|| > trans   OR  angle(R_last^T R) > rot.
 * R38: frame indices count from 0 (framesSinceStart = frame), framesSinceLastUpdate = frame - last;
 * the rotation distance is the angle of the relative rotation, acos((trace - 1) / 2). */
int oracle_should_recombine(int64_t frame, int64_t last, const double pose[16], const double last_pose[16],
                            int64_t boot, int64_t stale, double trans, double rot) {
  if (frame < boot) return 1;
  if (frame - last > stale) return 1;
  double dt[3] = {pose[3] - last_pose[3], pose[7] - last_pose[7], pose[11] - last_pose[11]};
  if (sqrt(dt[0] * dt[0] + dt[1] * dt[1] + dt[2] * dt[2]) > trans) return 1;
  double tr = 0.0; /* trace(R_last^T R) = sum_ab R_last[a][b] R[a][b] */
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) tr += last_pose[4 * a + b] * pose[4 * a + b];
  double cs = (tr - 1.0) / 2.0;
  cs = cs > 1.0 ? 1.0 : (cs < -1.0 ? -1.0 : cs);
  return acos(cs) > rot;
}
