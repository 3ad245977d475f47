/*
 * icp.c -- plain, slow, fp64 CPU reference of the weighted geometric point-to-plane ICP that
 * registers a depth frame against a rendered view.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.c).  Shares no code with the CUDA path.
 *
 * What it computes (readings R47-R52):
 *   association  frame pixel i with valid depth z -> camera point p_i (eq:reprojection P:532);
 *                x_i = DeltaT p_i in the rendered view's camera frame; projected to the nearest
 *                rendered pixel ("projective data association"); q_i, n_i = the rendered
 *                point and normal there (the renderer's world normal rotated into its camera frame)
 *   residual     r_i = <q_i - x_i, n_i> (eq:geometric_ICP at xi = 0), rejected when |r_i| exceeds
 *                the depth-outlier threshold; weight w_i = w_ICP(z) (eq:ICP_weight)
 *   Jacobian     J_i = (-n_i, -x_i x n_i) (eq:ICP_geometric_dx)
 *   normal eqs   H = 2 sum w_i J_i J_i^T, g = 2 sum w_i J_i r_i (eq:ICP_Hessian), summed in
 *                pixel order
 *   step         H xi = -g by Cholesky (eq:ICP_solution); DeltaT <- exp(xi) DeltaT
 *                (eq:deltaT_update); until |xi| < min_step or max_iters
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

typedef struct {
  double fx, fy, cx, cy, zmin, zmax;
  int W, H;
} icam;

static int z_ok(const icam *c, float z) { return z > 0.0f && (double)z >= c->zmin && (double)z <= c->zmax; }

/* 4x4 row-major products */
static void mat4_mul(const double A[16], const double B[16], double C[16]) {
  double T[16];
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      double s = 0.0;
      for (int k = 0; k < 4; ++k) s += A[4 * i + k] * B[4 * k + j];
      T[4 * i + j] = s;
    }
  memcpy(C, T, sizeof(T));
}

/* SE(3) exponential of xi = (nu, omega) (Blanco 2010, cited at P:276): R = Rodrigues(omega),
 * t = V(omega) nu with V = I + (1 - cos a)/a^2 W + (a - sin a)/a^3 W^2, W = [omega]_x */
void oracle_se3_exp(const double xi[6], double T[16]) {
  const double *nu = xi, *w = xi + 3;
  double a = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  double W[9] = {0, -w[2], w[1], w[2], 0, -w[0], -w[1], w[0], 0}, W2[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0.0;
      for (int k = 0; k < 3; ++k) s += W[3 * i + k] * W[3 * k + j];
      W2[3 * i + j] = s;
    }
  double A, B, Cc;
  if (a < 1e-8) { A = 1.0 - a * a / 6.0; B = 0.5 - a * a / 24.0; Cc = 1.0 / 6.0 - a * a / 120.0; }
  else { A = sin(a) / a; B = (1.0 - cos(a)) / (a * a); Cc = (a - sin(a)) / (a * a * a); }
  memset(T, 0, 16 * sizeof(double));
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) {
      double I = i == j ? 1.0 : 0.0;
      T[4 * i + j] = I + A * W[3 * i + j] + B * W2[3 * i + j];
    }
    double t = 0.0;
    for (int j = 0; j < 3; ++j) {
      double I = i == j ? 1.0 : 0.0;
      t += (I + B * W[3 * i + j] + Cc * W2[3 * i + j]) * nu[j];
    }
    T[4 * i + 3] = t;
  }
  T[15] = 1.0;
}

/*
 * Normal equations at DeltaT (eq:ICP_Hessian).  depth [H][W] the new frame; ref_depth [H][W]
 * and ref_normal [H][W][3] (world frame) the rendered view at ref_pose (world-from-camera);
 * intr fx fy cx cy W H zmin zmax.  Outputs H [36] (full), g [6], stats[0] inliers,
 * stats[1] sum w r^2.
 */
void oracle_icp_normal_equations(const float *depth, const float *ref_depth, const float *ref_normal,
                                 const double ref_pose[16], const double intr[8], const double delta[16],
                                 double outlier, double *Hout, double *gout, double *stats) {
  icam c = {intr[0], intr[1], intr[2], intr[3], intr[6], intr[7], (int)intr[4], (int)intr[5]};
  double H[36] = {0}, g[6] = {0}, cnt = 0.0, res = 0.0;
  for (int v = 0; v < c.H; ++v)
    for (int u = 0; u < c.W; ++u) {
      float z = depth[(size_t)v * c.W + u];
      if (!z_ok(&c, z)) continue;
      double p[3] = {((double)u - c.cx) / c.fx * (double)z, ((double)v - c.cy) / c.fy * (double)z, (double)z};
      double x[3];
      for (int a = 0; a < 3; ++a) x[a] = delta[4 * a] * p[0] + delta[4 * a + 1] * p[1] + delta[4 * a + 2] * p[2] + delta[4 * a + 3];
      if (!(x[2] > 0.0)) continue;
      double fu = floor(c.fx * x[0] / x[2] + c.cx + 0.5), fv = floor(c.fy * x[1] / x[2] + c.cy + 0.5);
      if (!(fu >= 0.0 && fu <= (double)(c.W - 1) && fv >= 0.0 && fv <= (double)(c.H - 1))) continue;
      int iu = (int)fu, iv = (int)fv;
      size_t j = (size_t)iv * c.W + iu;
      float zr = ref_depth[j];
      const float *nw = ref_normal + 3 * j;
      if (!z_ok(&c, zr) || (nw[0] == 0.0f && nw[1] == 0.0f && nw[2] == 0.0f)) continue;
      double q[3] = {((double)iu - c.cx) / c.fx * (double)zr, ((double)iv - c.cy) / c.fy * (double)zr, (double)zr};
      double n[3]; /* R_ref^T n_world */
      for (int a = 0; a < 3; ++a) n[a] = ref_pose[a] * nw[0] + ref_pose[4 + a] * nw[1] + ref_pose[8 + a] * nw[2];
      double r = (q[0] - x[0]) * n[0] + (q[1] - x[1]) * n[1] + (q[2] - x[2]) * n[2];
      if (!(fabs(r) <= outlier)) continue;
      double zz = (double)z + (1.0 - c.zmin);
      double w = 1.0 / (zz * zz); /* eq:ICP_weight */
      double xn[3] = {x[1] * n[2] - x[2] * n[1], x[2] * n[0] - x[0] * n[2], x[0] * n[1] - x[1] * n[0]};
      double J[6] = {-n[0], -n[1], -n[2], -xn[0], -xn[1], -xn[2]}; /* eq:ICP_geometric_dx */
      for (int a = 0; a < 6; ++a) {
        for (int b = 0; b < 6; ++b) H[6 * a + b] += 2.0 * w * J[a] * J[b];
        g[a] += 2.0 * w * J[a] * r;
      }
      cnt += 1.0;
      res += w * r * r;
    }
  memcpy(Hout, H, sizeof(H));
  memcpy(gout, g, sizeof(g));
  stats[0] = cnt;
  stats[1] = res;
}

/* Cholesky solve of H x = b (6x6, SPD); returns 0 or -1 when H is not positive definite */
int oracle_cholesky_solve6(const double Hin[36], const double b[6], double x[6]) {
  double L[36] = {0};
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = Hin[6 * i + j];
      for (int k = 0; k < j; ++k) s -= L[6 * i + k] * L[6 * j + k];
      if (i == j) {
        if (!(s > 0.0)) return -1;
        L[6 * i + i] = sqrt(s);
      } else {
        L[6 * i + j] = s / L[6 * j + j];
      }
    }
  double y[6];
  for (int i = 0; i < 6; ++i) {
    double s = b[i];
    for (int k = 0; k < i; ++k) s -= L[6 * i + k] * y[k];
    y[i] = s / L[6 * i + i];
  }
  for (int i = 5; i >= 0; --i) {
    double s = y[i];
    for (int k = i + 1; k < 6; ++k) s -= L[6 * k + i] * x[k];
    x[i] = s / L[6 * i + i];
  }
  return 0;
}

/* Gauss-Newton iterations from delta (in/out).  out[0] iterations, out[1] final step norm,
 * out[2] inliers of the last linearisation, out[3] its sum w r^2; returns 0, or -1 when the
 * system is singular (delta keeps the last good value). */
int oracle_icp(const float *depth, const float *ref_depth, const float *ref_normal, const double ref_pose[16],
               const double intr[8], double outlier, int max_iters, double min_step, double delta[16], double *out) {
  out[0] = out[1] = out[2] = out[3] = 0.0;
  for (int it = 0; it < max_iters; ++it) {
    double H[36], g[6], st[2], xi[6], mg[6];
    oracle_icp_normal_equations(depth, ref_depth, ref_normal, ref_pose, intr, delta, outlier, H, g, st);
    out[2] = st[0];
    out[3] = st[1];
    for (int a = 0; a < 6; ++a) mg[a] = -g[a];
    if (oracle_cholesky_solve6(H, mg, xi)) return -1;
    double E[16];
    oracle_se3_exp(xi, E);
    mat4_mul(E, delta, delta);
    double nrm = 0.0;
    for (int a = 0; a < 6; ++a) nrm += xi[a] * xi[a];
    out[0] = it + 1;
    out[1] = sqrt(nrm);
    if (out[1] < min_step) break;
  }
  return 0;
}
