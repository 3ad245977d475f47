/*
 * fusion.c -- plain, slow, fp64 CPU reference of voxel-projection fusion into the DTSDF
 * and of the depth-normal preprocessing it consumes.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.c): only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline legs may load it.  It shares no code with the CUDA path.
 *
 * What it computes (readings R39-R46):
 *   normals   n(u,v) = normalise((P(u+1,v) - P(u-1,v)) x (P(u,v+1) - P(u,v-1))), facing the camera
 *             ("Depth normals are approximated as cross product of neighboring pixels in x- and y
 *             direction"; the bilateral filter of that sentence is not applied, R39)
 *   allocate  for every valid pixel with world point p and world normal n, and every direction D
 *             with w_dir^D(n) > 0 (eq:angular_threshold), the blocks holding the
 *             points p + t n, t = -tau + j 2tau/M, j = 0..M, M = ceil(4 tau / s) (R40)
 *   fuse      every allocated voxel x of direction D projected into the frame (nearest pixel,
 *             "voxel projection"): d = <x - p, n> / tau (eq:point-to-plane,
 *             P:135-140, sign of reading R6: positive in front); d < -1 untouched; d > 1 free
 *             space: running average towards 1 with a constant weight, guarded by "no depth
 *             difference of more than tau in a radius of two pixels"; otherwise the
 *             weighted cumulative moving average with w_d = w_depth w_angle w_dir^D
 *             (eq:combined_fusion_weight; w_depth = w_ICP(z), eq:ICP_weight P:339,
 *             w_angle = <n, -ray>^+, R42) and the colour weight w_c = w_d (1 - min(1, |p-x|/tau))
 *             (eq:color_weight); weights capped at w_max (R44).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define FU_VPB 512

static const double FVDIR[6][3] = {{1, 0, 0}, {-1, 0, 0}, {0, 1, 0}, {0, -1, 0}, {0, 0, 1}, {0, 0, -1}};

typedef struct {
  double s, tau, theta, cos_theta;
  int64_t n, cap;
  int32_t *keys; /* [cap][4] */
  float *sdf, *w, *cw;
  uint8_t *rgb;
  int64_t hcap; /* open addressing over (packed location, direction) */
  uint64_t *hkey;
  int8_t *hdir;
  int64_t *hval;
} ofuse;

/* 3 x 21-bit block coordinates (63 bits); the direction is kept beside it */
static uint64_t fu_pack(int64_t x, int64_t y, int64_t z) {
  const uint64_t m = (1ull << 21) - 1;
  return ((uint64_t)(x + (1 << 20)) & m) | (((uint64_t)(y + (1 << 20)) & m) << 21) |
         (((uint64_t)(z + (1 << 20)) & m) << 42);
}

static int64_t fu_find(const ofuse *F, uint64_t k, int D) {
  uint64_t h = ((k + (uint64_t)D * 0x632BE59BD9B4E019ull) * 0x9E3779B97F4A7C15ull) >> 7;
  for (int64_t i = 0; i < F->hcap; ++i) {
    int64_t slot = (int64_t)((h + (uint64_t)i) % (uint64_t)F->hcap);
    if (F->hval[slot] < 0) return -1 - slot; /* free slot, encoded */
    if (F->hkey[slot] == k && F->hdir[slot] == D) return F->hval[slot];
  }
  return -1 - F->hcap;
}

static int64_t floordiv8(int64_t i) { return (i >= 0) ? i / 8 : -((-i + 7) / 8); }

/* returns 0, -1 bad key, -2 duplicate, -4 capacity */
static int fu_insert(ofuse *F, int64_t bx, int64_t by, int64_t bz, int64_t D, int init) {
  uint64_t k = fu_pack(bx, by, bz);
  int64_t r = fu_find(F, k, (int)D);
  if (r >= 0) return init ? -2 : 0;
  if (r == -1 - F->hcap || F->n >= F->cap) return -4;
  int64_t slot = -1 - r, b = F->n++;
  F->hkey[slot] = k;
  F->hdir[slot] = (int8_t)D;
  F->hval[slot] = b;
  F->keys[4 * b + 0] = (int32_t)bx; F->keys[4 * b + 1] = (int32_t)by;
  F->keys[4 * b + 2] = (int32_t)bz; F->keys[4 * b + 3] = (int32_t)D;
  if (!init)
    for (int l = 0; l < FU_VPB; ++l) { /* a new block: free space of weight 0 */
      F->sdf[b * FU_VPB + l] = 1.0f;
      F->w[b * FU_VPB + l] = 0.0f;
      F->cw[b * FU_VPB + l] = 0.0f;
      F->rgb[3 * (b * FU_VPB + l) + 0] = F->rgb[3 * (b * FU_VPB + l) + 1] = F->rgb[3 * (b * FU_VPB + l) + 2] = 0;
    }
  return 0;
}

void oracle_fuse_destroy(void *p) {
  ofuse *F = (ofuse *)p;
  if (!F) return;
  free(F->keys); free(F->sdf); free(F->w); free(F->cw); free(F->rgb); free(F->hkey); free(F->hdir); free(F->hval);
  free(F);
}

/* A fusion volume of capacity cap holding n0 initial blocks (keys/sdf/weight/rgb may be NULL if
 * n0 == 0); initial colour weights = the depth weights (R45).  Returns 0 or a negative code. */
int oracle_fuse_create(double s, double tau, double theta, int64_t cap, int64_t n0, const int32_t *keys,
                       const float *sdf, const float *weight, const uint8_t *rgb, void **out) {
  *out = NULL;
  if (cap < n0 || cap < 0) return -1;
  ofuse *F = (ofuse *)calloc(1, sizeof(ofuse));
  if (!F) return -4;
  F->s = s; F->tau = tau; F->theta = theta; F->cos_theta = cos(theta);
  F->cap = cap;
  size_t c = (size_t)(cap ? cap : 1);
  F->keys = (int32_t *)calloc(4 * c, sizeof(int32_t));
  F->sdf = (float *)calloc(c * FU_VPB, sizeof(float));
  F->w = (float *)calloc(c * FU_VPB, sizeof(float));
  F->cw = (float *)calloc(c * FU_VPB, sizeof(float));
  F->rgb = (uint8_t *)calloc(c * FU_VPB * 3, 1);
  F->hcap = 2 * (int64_t)c + 1;
  F->hkey = (uint64_t *)calloc((size_t)F->hcap, sizeof(uint64_t));
  F->hdir = (int8_t *)calloc((size_t)F->hcap, 1);
  F->hval = (int64_t *)malloc(sizeof(int64_t) * (size_t)F->hcap);
  if (!F->keys || !F->sdf || !F->w || !F->cw || !F->rgb || !F->hkey || !F->hdir || !F->hval) {
    oracle_fuse_destroy(F);
    return -4;
  }
  for (int64_t i = 0; i < F->hcap; ++i) F->hval[i] = -1;
  for (int64_t b = 0; b < n0; ++b) {
    if (keys[4 * b + 3] < 0 || keys[4 * b + 3] > 5) { oracle_fuse_destroy(F); return -1; }
    int rc = fu_insert(F, keys[4 * b], keys[4 * b + 1], keys[4 * b + 2], keys[4 * b + 3], 1);
    if (rc) { oracle_fuse_destroy(F); return rc; }
    memcpy(F->sdf + b * FU_VPB, sdf + b * FU_VPB, FU_VPB * sizeof(float));
    memcpy(F->w + b * FU_VPB, weight + b * FU_VPB, FU_VPB * sizeof(float));
    memcpy(F->cw + b * FU_VPB, weight + b * FU_VPB, FU_VPB * sizeof(float));
    if (rgb) memcpy(F->rgb + 3 * b * FU_VPB, rgb + 3 * b * FU_VPB, 3 * FU_VPB);
  }
  *out = F;
  return 0;
}

int64_t oracle_fuse_count(void *p) { return ((ofuse *)p)->n; }

/* copy out the first n blocks (n = oracle_fuse_count) */
void oracle_fuse_get(void *p, int32_t *keys, float *sdf, float *weight, uint8_t *rgb, float *cweight) {
  ofuse *F = (ofuse *)p;
  size_t n = (size_t)F->n;
  memcpy(keys, F->keys, n * 4 * sizeof(int32_t));
  memcpy(sdf, F->sdf, n * FU_VPB * sizeof(float));
  memcpy(weight, F->w, n * FU_VPB * sizeof(float));
  memcpy(rgb, F->rgb, n * FU_VPB * 3);
  if (cweight) memcpy(cweight, F->cw, n * FU_VPB * sizeof(float));
}

typedef struct {
  double R[9], t[3], fx, fy, cx, cy, zmin, zmax;
  int W, H;
} fcam;

static void fcam_from(fcam *c, const double pose[16], const double intr[8]) {
  for (int a = 0; a < 3; ++a) {
    for (int b = 0; b < 3; ++b) c->R[3 * a + b] = pose[4 * a + b];
    c->t[a] = pose[4 * a + 3];
  }
  c->fx = intr[0]; c->fy = intr[1]; c->cx = intr[2]; c->cy = intr[3];
  c->W = (int)intr[4]; c->H = (int)intr[5]; c->zmin = intr[6]; c->zmax = intr[7];
}

/* R41: a depth pixel is valid iff its depth lies in [zmin, zmax] (0 = missing) */
static int depth_ok(const fcam *c, float z) { return z > 0.0f && (double)z >= c->zmin && (double)z <= c->zmax; }

/* camera point of pixel (u, v) at depth z (eq:reprojection) */
static void backproject(const fcam *c, int u, int v, double z, double P[3]) {
  P[0] = ((double)u - c->cx) / c->fx * z;
  P[1] = ((double)v - c->cy) / c->fy * z;
  P[2] = z;
}

/* world = R P + t, each component ((R0 P0 + R1 P1) + R2 P2) + t, one rounding per operation */
static void to_world(const fcam *c, const double P[3], double X[3]) {
  for (int a = 0; a < 3; ++a) X[a] = c->R[3 * a] * P[0] + c->R[3 * a + 1] * P[1] + c->R[3 * a + 2] * P[2] + c->t[a];
}

static void rotate(const fcam *c, const double n[3], double m[3]) {
  for (int a = 0; a < 3; ++a) m[a] = c->R[3 * a] * n[0] + c->R[3 * a + 1] * n[1] + c->R[3 * a + 2] * n[2];
}

/* R39: camera-frame normals; out [H][W][3], 0 where invalid */
void oracle_depth_normals(const float *depth, const double intr[8], float *out) {
  fcam c;
  double pose[16] = {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1};
  fcam_from(&c, pose, intr);
  for (int v = 0; v < c.H; ++v)
    for (int u = 0; u < c.W; ++u) {
      float *o = out + 3 * ((size_t)v * c.W + u);
      o[0] = o[1] = o[2] = 0.0f;
      if (u < 1 || v < 1 || u >= c.W - 1 || v >= c.H - 1) continue;
      float zc = depth[(size_t)v * c.W + u], zl = depth[(size_t)v * c.W + u - 1], zr = depth[(size_t)v * c.W + u + 1];
      float zu = depth[(size_t)(v - 1) * c.W + u], zd = depth[(size_t)(v + 1) * c.W + u];
      if (!depth_ok(&c, zc) || !depth_ok(&c, zl) || !depth_ok(&c, zr) || !depth_ok(&c, zu) || !depth_ok(&c, zd)) continue;
      double P[3], L[3], Rr[3], U[3], D[3];
      backproject(&c, u, v, zc, P);
      backproject(&c, u - 1, v, zl, L);
      backproject(&c, u + 1, v, zr, Rr);
      backproject(&c, u, v - 1, zu, U);
      backproject(&c, u, v + 1, zd, D);
      double a[3] = {Rr[0] - L[0], Rr[1] - L[1], Rr[2] - L[2]}, b[3] = {D[0] - U[0], D[1] - U[1], D[2] - U[2]};
      double n[3] = {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
      double nn = sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
      if (!(nn > 0.0)) continue;
      double sgn = (n[0] * P[0] + n[1] * P[1] + n[2] * P[2]) > 0.0 ? -1.0 : 1.0; /* face the camera */
      for (int k = 0; k < 3; ++k) o[k] = (float)(sgn * n[k] / nn);
    }
}

static double fu_w_dir(double c, double theta) {
  double cc = c < -1.0 ? -1.0 : (c > 1.0 ? 1.0 : c);
  double w = (theta - acos(cc)) / (2.0 * theta - M_PI / 2.0);
  return w < 0.0 ? 0.0 : (w > 1.0 ? 1.0 : w);
}

static uint8_t fu_u8(double c) {
  double q = floor(c + 0.5);
  return (uint8_t)(q > 255.0 ? 255.0 : (q < 0.0 ? 0.0 : q));
}

/*
 * Allocate and fuse one frame.  depth [H][W] camera z (0 = missing), normal [H][W][3] unit
 * camera-frame normals facing the camera (0 = invalid), color [H][W][3] (may be NULL); pose
 * world-from-camera; intr fx fy cx cy W H zmin zmax; prm = {w_max, carve_weight, carve_radius}.
 * Returns the number of new blocks, or -4 when the capacity is exhausted (blocks allocated so
 * far are kept; the frame is not fused).
 */
int64_t oracle_fuse_frame(void *p, const float *depth, const float *normal, const uint8_t *color, const double pose[16],
                          const double intr[8], const double prm[3]) {
  ofuse *F = (ofuse *)p;
  fcam c;
  fcam_from(&c, pose, intr);
  const double wmax = prm[0], carve_w = prm[1];
  const int rad = (int)prm[2];
  const int64_t n_before = F->n;
  /* R40: allocation */
  const int M = (int)ceil(4.0 * F->tau / F->s);
  const double step = 2.0 * F->tau / (double)M;
  for (int v = 0; v < c.H; ++v)
    for (int u = 0; u < c.W; ++u) {
      size_t i = (size_t)v * c.W + u;
      const float *nc = normal + 3 * i;
      if (!depth_ok(&c, depth[i]) || (nc[0] == 0.0f && nc[1] == 0.0f && nc[2] == 0.0f)) continue;
      double P[3], X[3], n0[3] = {nc[0], nc[1], nc[2]}, n[3];
      backproject(&c, u, v, depth[i], P);
      to_world(&c, P, X);
      rotate(&c, n0, n);
      for (int D = 0; D < 6; ++D) {
        if (!(n[0] * FVDIR[D][0] + n[1] * FVDIR[D][1] + n[2] * FVDIR[D][2] > F->cos_theta)) continue;
        for (int j = 0; j <= M; ++j) {
          double tj = -F->tau + (double)j * step;
          int64_t b[3];
          for (int a = 0; a < 3; ++a) b[a] = floordiv8((int64_t)floor((X[a] + tj * n[a]) / F->s));
          if (fu_insert(F, b[0], b[1], b[2], D, 0) == -4) return -4;
        }
      }
    }
  /* R41-R45: voxel projection fusion of every allocated voxel */
  for (int64_t b = 0; b < F->n; ++b) {
    const int D = F->keys[4 * b + 3];
    for (int l = 0; l < FU_VPB; ++l) {
      int64_t vi[3] = {8 * (int64_t)F->keys[4 * b] + (l & 7), 8 * (int64_t)F->keys[4 * b + 1] + ((l >> 3) & 7),
                       8 * (int64_t)F->keys[4 * b + 2] + (l >> 6)};
      double x[3] = {(double)vi[0] * F->s, (double)vi[1] * F->s, (double)vi[2] * F->s};
      double d0[3] = {x[0] - c.t[0], x[1] - c.t[1], x[2] - c.t[2]}, xc[3];
      for (int a = 0; a < 3; ++a) xc[a] = c.R[a] * d0[0] + c.R[3 + a] * d0[1] + c.R[6 + a] * d0[2];
      if (!(xc[2] > 0.0)) continue;
      double uu = c.fx * xc[0] / xc[2] + c.cx, vv = c.fy * xc[1] / xc[2] + c.cy;
      double fu = floor(uu + 0.5), fv = floor(vv + 0.5); /* R41: nearest pixel */
      if (!(fu >= 0.0 && fu <= (double)(c.W - 1) && fv >= 0.0 && fv <= (double)(c.H - 1))) continue;
      int iu = (int)fu, iv = (int)fv;
      size_t pi = (size_t)iv * c.W + iu;
      const float *nc = normal + 3 * pi;
      float z = depth[pi];
      if (!depth_ok(&c, z) || (nc[0] == 0.0f && nc[1] == 0.0f && nc[2] == 0.0f)) continue;
      double P[3], X[3], n0[3] = {nc[0], nc[1], nc[2]}, n[3];
      backproject(&c, iu, iv, z, P);
      to_world(&c, P, X);
      rotate(&c, n0, n);
      double dd = ((x[0] - X[0]) * n[0] + (x[1] - X[1]) * n[1] + (x[2] - X[2]) * n[2]) / F->tau; /* R6 sign */
      size_t r = (size_t)b * FU_VPB + l;
      if (dd < -1.0) continue; /* behind the surface beyond the band: untouched */
      if (dd > 1.0) {
        /* R43: free space -> towards 1 with a constant weight, unless a depth within `rad`
         * pixels differs by more than tau (depth edge); a carving weight of 0 means no carving
         * (on a fresh voxel, W0 = 0, the running average would be 0/0) */
        if (!(carve_w > 0.0)) continue;
        int edge = 0;
        for (int dv = -rad; dv <= rad && !edge; ++dv)
          for (int du = -rad; du <= rad; ++du) {
            int qu = iu + du, qv = iv + dv;
            if (qu < 0 || qv < 0 || qu >= c.W || qv >= c.H) continue;
            float zq = depth[(size_t)qv * c.W + qu];
            if (!depth_ok(&c, zq)) continue;
            if (fabs((double)zq - (double)z) > F->tau) { edge = 1; break; }
          }
        if (edge) continue;
        double W0 = F->w[r];
        F->sdf[r] = (float)((W0 * (double)F->sdf[r] + carve_w * 1.0) / (W0 + carve_w));
        F->w[r] = (float)(W0 + carve_w < wmax ? W0 + carve_w : wmax);
        continue;
      }
      double wdir = fu_w_dir(n[0] * FVDIR[D][0] + n[1] * FVDIR[D][1] + n[2] * FVDIR[D][2], F->theta);
      double ray[3] = {X[0] - c.t[0], X[1] - c.t[1], X[2] - c.t[2]};
      double rl = sqrt(ray[0] * ray[0] + ray[1] * ray[1] + ray[2] * ray[2]);
      double ca = rl > 0.0 ? -(n[0] * ray[0] + n[1] * ray[1] + n[2] * ray[2]) / rl : 0.0;
      double wang = ca > 0.0 ? ca : 0.0;                                        /* R42 */
      double wdep = 1.0 / (((double)z + (1.0 - c.zmin)) * ((double)z + (1.0 - c.zmin))); /* eq:ICP_weight */
      double wn = wdep * wang * wdir;                                           /* eq:combined_fusion_weight */
      if (!(wn > 0.0)) continue;
      double W0 = F->w[r];
      F->sdf[r] = (float)((W0 * (double)F->sdf[r] + wn * dd) / (W0 + wn));
      F->w[r] = (float)(W0 + wn < wmax ? W0 + wn : wmax);
      if (color) {
        double dist = sqrt((X[0] - x[0]) * (X[0] - x[0]) + (X[1] - x[1]) * (X[1] - x[1]) + (X[2] - x[2]) * (X[2] - x[2]));
        double wc = wn * (1.0 - (dist / F->tau < 1.0 ? dist / F->tau : 1.0)); /* eq:color_weight */
        if (wc > 0.0) {
          double C0 = F->cw[r];
          for (int a = 0; a < 3; ++a)
            F->rgb[3 * r + a] = fu_u8((C0 * (double)F->rgb[3 * r + a] + wc * (double)color[3 * pi + a]) / (C0 + wc));
          F->cw[r] = (float)(C0 + wc < wmax ? C0 + wc : wmax);
        }
      }
    }
  }
  return F->n - n_before;
}
