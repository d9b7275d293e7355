// chain_common.cuh — per-chain device helpers shared by the per-chain kernels
// (kernels.cu, nuts.cu, ncp.cu): the heights map, block reductions, Philox,
// the torus spectrum.  Internal to libmt.
#pragma once
#include <math.h>

#include "mt_internal.cuh"

namespace {

constexpr double kTClamp = 10.0;  // R18

struct NodeH {
  float H0, H1;      // heights (fp32, computed in fp64)
  float L0, L1;      // fp32 residuals: H + L = the fp64 heights to ~1e-14 (HP2)
  double J0, J10, J11;  // ∂H0/∂x0, ∂H1/∂x0, ∂H1/∂x1
  double t0, t1;        // x/σ (clamped): ∂H/∂σ = -t·∂H/∂x (sampled r, f2)
};

// Gaussian copula + stick-breaking: ǔ = Φ(clamp(x/σ)),
// H0 = ǔ0 z_top, H1 = H0 + ǔ1 (z_top - H0).  fp64 internally (HP2 lever 2).
__device__ __forceinline__ NodeH node_heights(double x0, double x1, double is0, double is1,
                                              float z_top, bool want_jac) {
  NodeH o;
  double t0 = x0 * is0, t1 = x1 * is1;
  bool c0 = fabs(t0) > kTClamp, c1 = fabs(t1) > kTClamp;
  t0 = fmin(fmax(t0, -kTClamp), kTClamp);
  t1 = fmin(fmax(t1, -kTClamp), kTClamp);
  double u0 = 0.5 * erfc(-t0 * M_SQRT1_2), u1 = 0.5 * erfc(-t1 * M_SQRT1_2);
  double zt = (double)z_top;
  double h0 = u0 * zt, h1 = h0 + u1 * (zt - h0);
  o.H0 = (float)h0;
  o.H1 = (float)h1;
  o.L0 = (float)(h0 - (double)o.H0);
  o.L1 = (float)(h1 - (double)o.H1);
  o.t0 = t0;
  o.t1 = t1;
  if (want_jac) {
    const double inv_sqrt_2pi = 0.39894228040143267794;
    double d0 = c0 ? 0.0 : exp(-0.5 * t0 * t0) * inv_sqrt_2pi * is0;
    double d1 = c1 ? 0.0 : exp(-0.5 * t1 * t1) * inv_sqrt_2pi * is1;
    o.J0 = zt * d0;
    o.J10 = (1.0 - u1) * zt * d0;
    o.J11 = (zt - h0) * d1;
  }
  return o;
}

// The Jacobian of node_heights in fp32 (∂H0/∂x0, ∂H1/∂x0, ∂H1/∂x1): the chain rule
// needs it to fp32 accuracy only (the gradient's tolerance is 1e-3), unlike the
// heights themselves (HP2), so the group-tiled K3 spends no fp64 copula on it.
struct JacF {
  float J0, J10, J11;
};
__device__ __forceinline__ JacF node_jac32(float x0, float x1, double is0, double is1, float z_top) {
  const float s0 = (float)is0, s1 = (float)is1;
  float t0 = x0 * s0, t1 = x1 * s1;
  const bool c0 = fabsf(t0) > (float)kTClamp, c1 = fabsf(t1) > (float)kTClamp;
  t0 = fminf(fmaxf(t0, -(float)kTClamp), (float)kTClamp);
  t1 = fminf(fmaxf(t1, -(float)kTClamp), (float)kTClamp);
  const float u0 = 0.5f * erfcf(-t0 * 0.70710678118654752f), u1 = 0.5f * erfcf(-t1 * 0.70710678118654752f);
  const float inv_sqrt_2pi = 0.39894228040143268f;
  const float d0 = c0 ? 0.f : expf(-0.5f * t0 * t0) * inv_sqrt_2pi * s0;
  const float d1 = c1 ? 0.f : expf(-0.5f * t1 * t1) * inv_sqrt_2pi * s1;
  JacF j;
  j.J0 = z_top * d0;
  j.J10 = (1.f - u1) * z_top * d0;
  j.J11 = (z_top - u0 * z_top) * d1;
  return j;
}

// diagonal inverse mass M^-1 (mt_set_inverse_mass; identity when not set):
// p ~ N(0, M), drift x += ε M^-1 p, kinetic ½ pᵀ M^-1 p (R19b)
__device__ __forceinline__ float mi(const FinishArgs &a, int k) { return a.minv ? a.minv[k] : 1.f; }

__device__ __forceinline__ float warp_min(float v) {
  for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide reductions (256 threads): band min/max and up to 2 double sums.
struct BlockRed {
  float mn0, mx0, mn1, mx1;
  double s0, s1;
  int bad;
};

__device__ __forceinline__ BlockRed block_reduce(BlockRed v) {
  __shared__ float sh[4][MT_THREADS / 32];
  __shared__ double sd[2][MT_THREADS / 32];
  __shared__ int sb[MT_THREADS / 32];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v.mn0 = warp_min(v.mn0); v.mx0 = warp_max(v.mx0);
  v.mn1 = warp_min(v.mn1); v.mx1 = warp_max(v.mx1);
  v.s0 = warp_sum(v.s0); v.s1 = warp_sum(v.s1);
  v.bad = __any_sync(0xffffffffu, v.bad);
  if (lane == 0) {
    sh[0][w] = v.mn0; sh[1][w] = v.mx0; sh[2][w] = v.mn1; sh[3][w] = v.mx1;
    sd[0][w] = v.s0; sd[1][w] = v.s1; sb[w] = v.bad;
  }
  __syncthreads();
  BlockRed r = {3.0e38f, -3.0e38f, 3.0e38f, -3.0e38f, 0.0, 0.0, 0};
  if (threadIdx.x == 0) {
    for (int k = 0; k < nw; k++) {
      r.mn0 = fminf(r.mn0, sh[0][k]); r.mx0 = fmaxf(r.mx0, sh[1][k]);
      r.mn1 = fminf(r.mn1, sh[2][k]); r.mx1 = fmaxf(r.mx1, sh[3][k]);
      r.s0 += sd[0][k]; r.s1 += sd[1][k]; r.bad |= sb[k];
    }
  }
  return r;  // valid in thread 0
}

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al. SC'11), the counter-based generator of R22.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint4 philox10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; r++) {
    uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

__device__ __forceinline__ double u01(uint32_t w) { return ((double)w + 0.5) * 2.3283064365386963e-10; }

// Momenta for parameters 4q..4q+3 of global chain `chain` (Box-Muller, fp64).
__device__ __forceinline__ void momenta4(uint64_t seed, uint64_t iter, uint64_t chain, int q,
                                         double z[4]) {
  uint4 w = philox10(make_uint4((uint32_t)q, (uint32_t)chain, (uint32_t)iter, 0u),
                     make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
  uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int h = 0; h < 2; h++) {
    double rad = sqrt(-2.0 * log(u01(ww[2 * h])));
    double sn, cs;
    sincospi(2.0 * u01(ww[2 * h + 1]), &sn, &cs);
    z[2 * h] = rad * cs;
    z[2 * h + 1] = rad * sn;
  }
}

// ---------------------------------------------------------------------------
// Sampled r_l (readings R13b/R13c): state per chain
// (x_0, x_1, ρ_0, ρ_1), r_l = logistic(ρ_l).  Every per-chain kernel first
// evaluates the torus spectrum of Q(r_l) = 4I - r_l A for its chain (a block
// reduction over the N eigenvalues λ = 4 - r c_ab, c_ab = 2(cos 2πa/n_x +
// cos 2πb/n_y)): σ_l (the copula scale), dσ_l/dr, ln det Q(r_l)
// and its derivative.
// ---------------------------------------------------------------------------
// In-place block sum of K doubles (all threads get the totals).
template <int K>
__device__ __forceinline__ void block_sum(double *v) {
  __shared__ double sh[K][MT_THREADS / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int q = 0; q < K; q++) v[q] = warp_sum(v[q]);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < K; q++) sh[q][w] = v[q];
  __syncthreads();
#pragma unroll
  for (int q = 0; q < K; q++) {
    double t = 0.0;
    for (int k = 0; k < nw; k++) t += sh[q][k];
    v[q] = t;
  }
  __syncthreads();
}

struct Spec {
  double r[2], inv_sigma[2], dsig[2], ld[2], dld[2];
};

__device__ __forceinline__ Spec block_spectrum(const double *cs, int N, float rho0, float rho1, bool logs) {
  Spec o;
  o.r[0] = 1.0 / (1.0 + exp(-(double)rho0));
  o.r[1] = 1.0 / (1.0 + exp(-(double)rho1));
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    const double c = cs[k];
#pragma unroll
    for (int l = 0; l < 2; l++) {
      const double lam = 4.0 - o.r[l] * c, il = 1.0 / lam;
      acc[4 * l] += il;
      acc[4 * l + 1] += c * il * il;
      if (logs) acc[4 * l + 2] += log(lam);
      acc[4 * l + 3] -= c * il;
    }
  }
  block_sum<8>(acc);
#pragma unroll
  for (int l = 0; l < 2; l++) {
    const double sg = sqrt(acc[4 * l] / N);
    o.inv_sigma[l] = 1.0 / sg;
    o.dsig[l] = (acc[4 * l + 1] / N) / (2.0 * sg);
    o.ld[l] = acc[4 * l + 2];
    o.dld[l] = acc[4 * l + 3];
  }
  return o;
}

}  // namespace
