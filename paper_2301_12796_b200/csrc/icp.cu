// icp.cu -- weighted geometric point-to-plane ICP of a depth frame against a rendered view with a
// deterministic reduction.
//
//   k_icp_reduce   fixed pixel -> thread mapping (DTSDF_ICP_PIX = 5 pixels per thread, 1280 per CTA): projective
//                  association of DeltaT p into the rendered view (fp64, the oracle's roundings,
//                  so both sides associate the same pixels), r = <q - x, n>, J = (-n, -x x n),
//                  w = w_ICP(z); the 21 + 6 + 2 sums (upper H, g, inliers, sum w r^2) in fp64, reduced
//                  by a fixed shuffle tree per warp and a fixed warp order per CTA -> one partial per
//                  CTA ("fully-deterministic hierarchical scheme")
//   k_icp_solve    one CTA: the partials reduced in a fixed order, H xi = -g by Cholesky,
//                  DeltaT <- exp(xi) DeltaT, termination on |xi| < min_step or the iteration
//                  cap; sets the done flag that turns the remaining launches into no-ops
//
// Iterations are enqueued in chunks (2 launches each); the host polls the done flag between chunks.
#include "common.cuh"

namespace dtsdf {

#ifndef DTSDF_ICP_PIX
#define DTSDF_ICP_PIX 5  // 1280 pixels per CTA: a 640x480 frame is 240 CTAs, one wave of 2 per SM (4 gave 300: 4 CTAs in a 2nd wave)
#endif
constexpr int kIcpThreads = 256, kIcpPix = DTSDF_ICP_PIX, kIcpSums = 29;
#ifndef DTSDF_ICP_UNROLL
#define DTSDF_ICP_UNROLL 1
#endif
constexpr int kIcpUnroll = DTSDF_ICP_UNROLL;  // pixels of a thread in flight together

__device__ __forceinline__ bool icp_z_ok(const IcpLaunch &p, float z) {
  return z > 0.0f && (double)z >= p.z_min && (double)z <= p.z_max;
}

__device__ __forceinline__ void icp_pixel(const IcpLaunch &p, const double *D, int pix, double acc[kIcpSums]) {
  const float z = p.depth[pix];
  if (!icp_z_ok(p, z)) return;
  const double zd = (double)z;
  // the frame point's back-projection, computed once per call (k_icp_backproject, same operations)
  const double2 pb = p.pback[pix];
  const double p0 = pb.x, p1 = pb.y;
  double x[3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
    x[a] = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(D[4 * a], p0), __dmul_rn(D[4 * a + 1], p1)), __dmul_rn(D[4 * a + 2], zd)),
                     D[4 * a + 3]);
  if (!(x[2] > 0.0)) return;
  const double fu = floor(__dadd_rn(__dadd_rn(__ddiv_rn(__dmul_rn(p.fx, x[0]), x[2]), p.cx), 0.5));
  const double fv = floor(__dadd_rn(__dadd_rn(__ddiv_rn(__dmul_rn(p.fy, x[1]), x[2]), p.cy), 0.5));
  if (!(fu >= 0.0 && fu <= (double)(p.width - 1) && fv >= 0.0 && fv <= (double)(p.height - 1))) return;
  const int iu = (int)fu, iv = (int)fv;
  const size_t j = (size_t)iv * p.width + iu;
  DTSDF_CHECK(iu >= 0 && iu < p.width && iv >= 0 && iv < p.height);
  const float zr = p.ref_depth[j];
  const float nw0 = p.ref_normal[3 * j], nw1 = p.ref_normal[3 * j + 1], nw2 = p.ref_normal[3 * j + 2];
  if (!icp_z_ok(p, zr) || (nw0 == 0.f && nw1 == 0.f && nw2 == 0.f)) return;
  const double zrd = (double)zr;
  const double q0 = __dmul_rn(p.col_fac[iu], zrd);  // (iu - cx) / fx * zr, the factor tabulated per column
  const double q1 = __dmul_rn(p.row_fac[iv], zrd);
  double n[3];  // R_ref^T n_world
#pragma unroll
  for (int a = 0; a < 3; ++a)
    n[a] = __dadd_rn(__dadd_rn(__dmul_rn(p.ref_R[a], (double)nw0), __dmul_rn(p.ref_R[3 + a], (double)nw1)),
                     __dmul_rn(p.ref_R[6 + a], (double)nw2));
  const double r = __dadd_rn(__dadd_rn(__dmul_rn(__dsub_rn(q0, x[0]), n[0]), __dmul_rn(__dsub_rn(q1, x[1]), n[1])),
                             __dmul_rn(__dsub_rn(zrd, x[2]), n[2]));
  if (!(fabs(r) <= p.outlier)) return;  // depth outlier
  const double zz = zd + (1.0 - p.z_min);
  const double w2 = 2.0 / (zz * zz);  // 2 w_ICP(z) (eq:ICP_weight, eq:ICP_Hessian)
  const double J[6] = {-n[0], -n[1], -n[2], -(x[1] * n[2] - x[2] * n[1]), -(x[2] * n[0] - x[0] * n[2]),
                       -(x[0] * n[1] - x[1] * n[0])};
  int k = 0;
#pragma unroll
  for (int a = 0; a < 6; ++a)
#pragma unroll
    for (int b = a; b < 6; ++b) acc[k++] += w2 * J[a] * J[b];
#pragma unroll
  for (int a = 0; a < 6; ++a) acc[21 + a] += w2 * J[a] * r;
  acc[27] += 1.0;
  acc[28] += 0.5 * w2 * r * r;
}

// Per call: the frame's back-projected points (they do not change between iterations) and the
// per-column / per-row factors of the rendered pixels' back-projection -- the divisions of
// icp_pixel hoisted out of the iteration loop with the oracle's operations and roundings.
__global__ void k_icp_backproject(const __grid_constant__ IcpLaunch p) {
  const int pix = blockIdx.x * blockDim.x + threadIdx.x;
  if (pix < p.width) p.col_fac[pix] = __ddiv_rn(__dsub_rn((double)pix, p.cx), p.fx);
  if (pix < p.height) p.row_fac[pix] = __ddiv_rn(__dsub_rn((double)pix, p.cy), p.fy);
  if (pix >= p.width * p.height) return;
  const int u = pix % p.width, v = pix / p.width;
  const double zd = (double)p.depth[pix];
  p.pback[pix] = make_double2(__dmul_rn(__ddiv_rn(__dsub_rn((double)u, p.cx), p.fx), zd),
                              __dmul_rn(__ddiv_rn(__dsub_rn((double)v, p.cy), p.fy), zd));
}

__device__ void icp_solve_body(const IcpLaunch &p, int n_partials);

__global__ void __launch_bounds__(kIcpThreads) k_icp_reduce(const __grid_constant__ IcpLaunch p) {
  if (*((volatile int *)&p.state->done)) return;
  __shared__ double s_d[16];
  __shared__ double s_w[kIcpThreads / 32][kIcpSums];
  const int tid = threadIdx.x;
  if (tid < 16) s_d[tid] = p.state->delta[tid];
  __syncthreads();
  double acc[kIcpSums];
#pragma unroll
  for (int k = 0; k < kIcpSums; ++k) acc[k] = 0.0;
  const int npix = p.width * p.height;
#pragma unroll kIcpUnroll
  for (int k = 0; k < kIcpPix; ++k) {
    const int pix = blockIdx.x * (kIcpThreads * kIcpPix) + k * kIcpThreads + tid;
    if (pix < npix) icp_pixel(p, s_d, pix, acc);
  }
  // fixed shuffle tree within the warp, then the 8 warp sums in warp order
#pragma unroll
  for (int k = 0; k < kIcpSums; ++k) {
    double v = acc[k];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    if ((tid & 31) == 0) s_w[tid >> 5][k] = v;
  }
  __syncthreads();
  if (tid < kIcpSums) {
    double v = s_w[0][tid];
#pragma unroll
    for (int w = 1; w < kIcpThreads / 32; ++w) v += s_w[w][tid];
    p.partials[(size_t)blockIdx.x * kIcpSums + tid] = v;
  }
  if (!p.fused_solve) return;
  // the last CTA to finish this iteration solves it (one launch per iteration instead of two)
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(&p.state->ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  icp_solve_body(p, gridDim.x);
  if (tid == 0) p.state->ticket = 0;
}

__device__ void se3_exp(const double xi[6], double T[16]) {
  const double *nu = xi, *w = xi + 3;
  const double a = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  const double W[9] = {0, -w[2], w[1], w[2], 0, -w[0], -w[1], w[0], 0};
  double W2[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) W2[3 * i + j] = W[3 * i] * W[j] + W[3 * i + 1] * W[3 + j] + W[3 * i + 2] * W[6 + j];
  double A, B, C;
  if (a < 1e-8) {
    A = 1.0 - a * a / 6.0; B = 0.5 - a * a / 24.0; C = 1.0 / 6.0 - a * a / 120.0;
  } else {
    A = sin(a) / a; B = (1.0 - cos(a)) / (a * a); C = (a - sin(a)) / (a * a * a);
  }
  for (int i = 0; i < 3; ++i) {
    double t = 0.0;
    for (int j = 0; j < 3; ++j) {
      const double I = i == j ? 1.0 : 0.0;
      T[4 * i + j] = I + A * W[3 * i + j] + B * W2[3 * i + j];
      t += (I + B * W[3 * i + j] + C * W2[3 * i + j]) * nu[j];
    }
    T[4 * i + 3] = t;
  }
  T[12] = T[13] = T[14] = 0.0;
  T[15] = 1.0;
}

// The partials' sum (thread t adds partials t, t + 256, ... in order, then the fixed warp / CTA tree:
// the same bits whichever CTA runs it), the 6x6 solve and the DeltaT update.  All kIcpThreads threads.
__device__ void icp_solve_body(const IcpLaunch &p, int n_partials) {
  IcpState *st = p.state;
  __shared__ double s_sum[kIcpThreads / 32][kIcpSums];
  const int tid = threadIdx.x;
  // thread t sums partials t, t + 256, ... in order; then the fixed warp / CTA tree
  double acc[kIcpSums];
#pragma unroll
  for (int k = 0; k < kIcpSums; ++k) acc[k] = 0.0;
  for (int i = tid; i < n_partials; i += kIcpThreads)
#pragma unroll
    for (int k = 0; k < kIcpSums; ++k) acc[k] += __ldcg(&p.partials[(size_t)i * kIcpSums + k]);
#pragma unroll
  for (int k = 0; k < kIcpSums; ++k) {
    double v = acc[k];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    if ((tid & 31) == 0) s_sum[tid >> 5][k] = v;
  }
  __syncthreads();
  if (tid != 0) return;
  double S[kIcpSums];
  for (int k = 0; k < kIcpSums; ++k) {
    double v = s_sum[0][k];
    for (int w = 1; w < kIcpThreads / 32; ++w) v += s_sum[w][k];
    S[k] = v;
  }
  for (int k = 0; k < kIcpSums; ++k) st->sums[k] = S[k];
  double H[36];
  int k = 0;
  for (int a = 0; a < 6; ++a)
    for (int b = a; b < 6; ++b) { H[6 * a + b] = S[k]; H[6 * b + a] = S[k]; ++k; }
  // Cholesky H = L L^T, then L y = -g, L^T xi = y
  double L[36];
  for (int i = 0; i < 36; ++i) L[i] = 0.0;
  bool ok = true;
  for (int i = 0; i < 6 && ok; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = H[6 * i + j];
      for (int m = 0; m < j; ++m) s -= L[6 * i + m] * L[6 * j + m];
      if (i == j) {
        if (!(s > 0.0)) { ok = false; break; }
        L[6 * i + i] = sqrt(s);
      } else {
        L[6 * i + j] = s / L[6 * j + j];
      }
    }
  st->inliers = (long long)S[27];
  st->residual = S[28];
  if (!ok) {
    st->status = 1;  // singular: DeltaT keeps its last value
    st->done = 1;
    return;
  }
  double y[6], xi[6];
  for (int i = 0; i < 6; ++i) {
    double s = -S[21 + i];
    for (int m = 0; m < i; ++m) s -= L[6 * i + m] * y[m];
    y[i] = s / L[6 * i + i];
  }
  for (int i = 5; i >= 0; --i) {
    double s = y[i];
    for (int m = i + 1; m < 6; ++m) s -= L[6 * m + i] * xi[m];
    xi[i] = s / L[6 * i + i];
  }
  double E[16], Dn[16];
  se3_exp(xi, E);
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      double s = 0.0;
      for (int m = 0; m < 4; ++m) s += E[4 * i + m] * st->delta[4 * m + j];
      Dn[4 * i + j] = s;
    }
  for (int i = 0; i < 16; ++i) st->delta[i] = Dn[i];
  double nrm = 0.0;
  for (int i = 0; i < 6; ++i) nrm += xi[i] * xi[i];
  st->step = sqrt(nrm);
  st->iterations += 1;
  if (st->step < p.min_step || st->iterations >= p.max_iters) st->done = 1;
}

__global__ void __launch_bounds__(kIcpThreads) k_icp_solve(const __grid_constant__ IcpLaunch p, int n_partials) {
  if (*((volatile int *)&p.state->done)) return;
  icp_solve_body(p, n_partials);
}

int icp_partials(int width, int height) {
  return (width * height + kIcpThreads * kIcpPix - 1) / (kIcpThreads * kIcpPix);
}

cudaError_t launch_icp_backproject(const IcpLaunch &p, cudaStream_t s) {
  const int n = max(p.width * p.height, max(p.width, p.height));
  k_icp_backproject<<<(n + 255) / 256, 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_icp_reduce(const IcpLaunch &p, cudaStream_t s) {
  k_icp_reduce<<<icp_partials(p.width, p.height), kIcpThreads, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_icp_solve(const IcpLaunch &p, cudaStream_t s) {
  k_icp_solve<<<1, kIcpThreads, 0, s>>>(p, icp_partials(p.width, p.height));
  return cudaGetLastError();
}

}  // namespace dtsdf
