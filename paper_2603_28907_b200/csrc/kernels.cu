// kernels.cu — K1 (latent -> heights), K3 (chain rule + CAR prior + logpost,
// fused leapfrog kick/drift + next heights), HMC begin/end (Philox momenta,
// Metropolis), raw Philox, FP32 peak microbenchmark.  B200 / sm_100a.
//
// All per-chain kernels use one 256-thread block per chain: a chain's state is
// P = 2 n_x n_y <= 8192 floats, so a block streams it once (coalesced), does
// the 5-point periodic stencil from shared memory and reduces per-chain
// scalars without atomics.
#include <cooperative_groups.h>
#include <curand_philox4x32_x.h>
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

// ---------------------------------------------------------------------------
// K1: heights + per-chain band (min/max of each surface's node heights)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(MT_THREADS) k_heights(FinishArgs a, const float *x) {
  int c = blockIdx.x;
  const float *xc = x + (size_t)c * a.P;
  BlockRed v = {3.0e38f, -3.0e38f, 3.0e38f, -3.0e38f, 0.0, 0.0, 0};
  for (int k = threadIdx.x; k < a.N; k += blockDim.x) {
    NodeH h = node_heights(xc[k], xc[a.N + k], a.inv_sigma[0], a.inv_sigma[1], a.z_top, false);
    a.H[tix(c, 0, k, a.N)] = h.H0;
    a.H[tix(c, 1, k, a.N)] = h.H1;
    a.Hlo[tix(c, 0, k, a.N)] = h.L0;
    a.Hlo[tix(c, 1, k, a.N)] = h.L1;
    v.mn0 = fminf(v.mn0, h.H0); v.mx0 = fmaxf(v.mx0, h.H0);
    v.mn1 = fminf(v.mn1, h.H1); v.mx1 = fmaxf(v.mx1, h.H1);
  }
  BlockRed r = block_reduce(v);
  if (threadIdx.x == 0) a.band[c] = make_float4(r.mn0, r.mx0, r.mn1, r.mx1);
}

// ---------------------------------------------------------------------------
// K3: ∂ℓ/∂H -> ∂/∂x by the chain rule, CAR prior value and gradient (5-point
// periodic stencil), logpost assembly (fp64), and in
// leapfrog mode the fused kick / drift / next-heights update.
// ---------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(MT_THREADS) k_finish(FinishArgs a) {
  extern __shared__ float xs[];  // [2N] current x of this chain
  const int c = blockIdx.x, N = a.N, ny = a.ny, nx = a.nx;
  float *xc = a.x + (size_t)c * a.P;
  for (int k = threadIdx.x; k < a.P; k += blockDim.x) xs[k] = xc[k];
  __syncthreads();
  float *Gt = const_cast<float *>(a.G);
  float *gc = a.grad + (size_t)c * a.P;
  float *pc = MODE != FIN_PLAIN ? a.mom + (size_t)c * a.P : nullptr;
  const float eps = MODE != FIN_PLAIN ? a.eps[c] : 0.f;
  BlockRed v = {3.0e38f, -3.0e38f, 3.0e38f, -3.0e38f, 0.0, 0.0, 0};
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    const int i = k / ny, j = k - i * ny;
    float x0 = xs[k], x1 = xs[N + k];
    NodeH h = node_heights(x0, x1, a.inv_sigma[0], a.inv_sigma[1], a.z_top, true);
    const size_t t0 = tix(c, 0, k, N), t1 = tix(c, 1, k, N);
    float G0 = Gt[t0], G1 = Gt[t1];
    Gt[t0] = 0.f;
    Gt[t1] = 0.f;
    double gx0 = (double)G0 * h.J0 + (double)G1 * h.J10;
    double gx1 = (double)G1 * h.J11;
    if (a.prior_on) {
      const int ip = (i + 1 == nx ? 0 : i + 1) * ny + j, im = (i == 0 ? nx - 1 : i - 1) * ny + j;
      const int jp = i * ny + (j + 1 == ny ? 0 : j + 1), jm = i * ny + (j == 0 ? ny - 1 : j - 1);
#pragma unroll
      for (int l = 0; l < 2; l++) {
        const float *xl = xs + l * N;
        double xv = xl[k];
        double Qx = 4.0 * xv - (double)a.car_r[l] * ((double)xl[ip] + xl[im] + xl[jp] + xl[jm]);
        v.s0 += xv * Qx;
        if (l == 0) gx0 -= Qx; else gx1 -= Qx;
      }
    }
    float g0f = (float)gx0, g1f = (float)gx1;
    gc[k] = g0f;
    gc[N + k] = g1f;
    v.bad |= !(isfinite(g0f) && isfinite(g1f));
    if (MODE == FIN_STEP) {  // close this step's half kick, open the next: p += ε g; x += ε p
      float p0 = pc[k] + eps * g0f, p1 = pc[N + k] + eps * g1f;
      pc[k] = p0;
      pc[N + k] = p1;
      float xn0 = x0 + eps * mi(a, k) * p0, xn1 = x1 + eps * mi(a, N + k) * p1;
      xc[k] = xn0;
      xc[N + k] = xn1;
      NodeH hn = node_heights(xn0, xn1, a.inv_sigma[0], a.inv_sigma[1], a.z_top, false);
      a.H[t0] = hn.H0;
      a.H[t1] = hn.H1;
      a.Hlo[t0] = hn.L0;
      a.Hlo[t1] = hn.L1;
      v.mn0 = fminf(v.mn0, hn.H0); v.mx0 = fmaxf(v.mx0, hn.H0);
      v.mn1 = fminf(v.mn1, hn.H1); v.mx1 = fmaxf(v.mx1, hn.H1);
    } else if (MODE == FIN_LAST) {  // final half kick
      float p0 = pc[k] + 0.5f * eps * g0f, p1 = pc[N + k] + 0.5f * eps * g1f;
      pc[k] = p0;
      pc[N + k] = p1;
      v.s1 += 0.5 * ((double)mi(a, k) * p0 * p0 + (double)mi(a, N + k) * p1 * p1);
    }
  }
  BlockRed r = block_reduce(v);
  if (threadIdx.x == 0) {
    double lp = a.ll[c] + (a.prior_on ? -0.5 * r.s0 + a.prior_const : 0.0);
    a.ll[c] = 0.0;
    a.logp[c] = lp;
    int bad = r.bad || !isfinite(lp);
    if (a.status) a.status[c] = bad ? MT_STATUS_NONFINITE : 0;
    if (MODE == FIN_STEP) a.band[c] = make_float4(r.mn0, r.mx0, r.mn1, r.mx1);
    if (MODE == FIN_LAST && a.kin) a.kin[c] = (float)r.s1;
  }
}

// Leapfrog kicks from a stored gradient (R19):
//   KICK_HALF_DRIFT  p += ε/2 g; x += ε p; H(x)   (first step of mt_leapfrog)
//   KICK_FULL_DRIFT  p += ε g;   x += ε p; H(x)   (ray sharding: after the all-reduce)
//   KICK_HALF_LAST   p += ε/2 g; kinetic ½|p|²     (ray sharding: last step)
// The arithmetic is k_finish<FIN_STEP / FIN_LAST>'s, so a one-rank
// communicator reproduces the unsharded trajectory exactly.
template <int MODE>
__global__ void __launch_bounds__(MT_THREADS) k_kick(FinishArgs a) {
  const int c = blockIdx.x, N = a.N;
  float *xc = a.x + (size_t)c * a.P, *pc = a.mom + (size_t)c * a.P;
  const float *gc = a.grad + (size_t)c * a.P;
  const float eps = a.eps[c];
  const float f = MODE == KICK_FULL_DRIFT ? eps : 0.5f * eps;
  BlockRed v = {3.0e38f, -3.0e38f, 3.0e38f, -3.0e38f, 0.0, 0.0, 0};
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    float p0 = pc[k] + f * gc[k], p1 = pc[N + k] + f * gc[N + k];
    pc[k] = p0;
    pc[N + k] = p1;
    if (MODE == KICK_HALF_LAST) {
      v.s1 += 0.5 * ((double)mi(a, k) * p0 * p0 + (double)mi(a, N + k) * p1 * p1);
      continue;
    }
    float x0 = xc[k] + eps * mi(a, k) * p0, x1 = xc[N + k] + eps * mi(a, N + k) * p1;
    xc[k] = x0;
    xc[N + k] = x1;
    NodeH h = node_heights(x0, x1, a.inv_sigma[0], a.inv_sigma[1], a.z_top, false);
    a.H[tix(c, 0, k, N)] = h.H0;
    a.H[tix(c, 1, k, N)] = h.H1;
    a.Hlo[tix(c, 0, k, N)] = h.L0;
    a.Hlo[tix(c, 1, k, N)] = h.L1;
    v.mn0 = fminf(v.mn0, h.H0); v.mx0 = fmaxf(v.mx0, h.H0);
    v.mn1 = fminf(v.mn1, h.H1); v.mx1 = fmaxf(v.mx1, h.H1);
  }
  BlockRed r = block_reduce(v);
  if (threadIdx.x == 0) {
    if (MODE == KICK_HALF_LAST) a.kin[c] = (float)r.s1;
    else a.band[c] = make_float4(r.mn0, r.mx0, r.mn1, r.mx1);
  }
}

// ---------------------------------------------------------------------------
// Few chains (C < 16, e.g. the one-chain ray-sharded config): one block per
// chain leaves 147 of 148 SMs idle in K3 (68 µs of a 0.49 ms evaluation at
// N = 4096).  These variants spread a chain's nodes over gridDim.y blocks;
// the per-chain scalars go through fp64 atomics into a small scratch record,
// and the last block of the chain (atomic ticket) finalises and resets it.
// The leapfrog then runs unfused (K3 PLAIN + kick/drift), so no block reads a
// neighbour's x while another block drifts it.
// scratch per chain: red[0] Σ x·Qx, red[1] kinetic, red[2] non-finite flag,
//   bandi[4] = (min H0, max H0, min H1, max H1) as ordered float bits (heights >= 0)
// ---------------------------------------------------------------------------
struct MbScratch {
  double *red;          // [C][3]
  unsigned *bandi;      // [C][4]
  unsigned *ticket;     // [C]
};

__device__ __forceinline__ bool mb_last(unsigned *ticket, int c) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket + c, 1u) == gridDim.y - 1;
  __syncthreads();
  return last;
}

__global__ void __launch_bounds__(MT_THREADS) k_finish_mb(FinishArgs a, MbScratch m) {
  const int c = blockIdx.x, N = a.N, ny = a.ny, nx = a.nx;
  const float *xc = a.x + (size_t)c * a.P;
  float *gc = a.grad + (size_t)c * a.P;
  float *Gt = const_cast<float *>(a.G);
  BlockRed v = {3.0e38f, -3.0e38f, 3.0e38f, -3.0e38f, 0.0, 0.0, 0};
  for (int k = blockIdx.y * blockDim.x + threadIdx.x; k < N; k += gridDim.y * blockDim.x) {
    const int i = k / ny, j = k - i * ny;
    const float x0 = xc[k], x1 = xc[N + k];
    const NodeH h = node_heights(x0, x1, a.inv_sigma[0], a.inv_sigma[1], a.z_top, true);
    const size_t t0 = tix(c, 0, k, N), t1 = tix(c, 1, k, N);
    const float G0 = Gt[t0], G1 = Gt[t1];
    Gt[t0] = 0.f;
    Gt[t1] = 0.f;
    double gx0 = (double)G0 * h.J0 + (double)G1 * h.J10;
    double gx1 = (double)G1 * h.J11;
    if (a.prior_on) {
      const int ip = (i + 1 == nx ? 0 : i + 1) * ny + j, im = (i == 0 ? nx - 1 : i - 1) * ny + j;
      const int jp = i * ny + (j + 1 == ny ? 0 : j + 1), jm = i * ny + (j == 0 ? ny - 1 : j - 1);
#pragma unroll
      for (int l = 0; l < 2; l++) {
        const float *xl = xc + l * N;
        const double xv = xl[k];
        const double Qx = 4.0 * xv - (double)a.car_r[l] * ((double)xl[ip] + xl[im] + xl[jp] + xl[jm]);
        v.s0 += xv * Qx;
        if (l == 0) gx0 -= Qx; else gx1 -= Qx;
      }
    }
    const float g0f = (float)gx0, g1f = (float)gx1;
    gc[k] = g0f;
    gc[N + k] = g1f;
    v.bad |= !(isfinite(g0f) && isfinite(g1f));
  }
  const BlockRed r = block_reduce(v);
  if (threadIdx.x == 0) {
    atomicAdd(m.red + 3 * c, r.s0);
    if (r.bad) atomicAdd(m.red + 3 * c + 2, 1.0);
  }
  if (mb_last(m.ticket, c) && threadIdx.x == 0) {
    volatile double *rd = m.red + 3 * c;
    const double lp = a.ll[c] + (a.prior_on ? -0.5 * rd[0] + a.prior_const : 0.0);
    a.ll[c] = 0.0;
    a.logp[c] = lp;
    if (a.status) a.status[c] = (rd[2] != 0.0 || !isfinite(lp)) ? MT_STATUS_NONFINITE : 0;
    rd[0] = 0.0;
    rd[2] = 0.0;
    m.ticket[c] = 0u;
  }
}

template <int MODE>
__global__ void __launch_bounds__(MT_THREADS) k_kick_mb(FinishArgs a, MbScratch m) {
  const int c = blockIdx.x, N = a.N;
  float *xc = a.x + (size_t)c * a.P, *pc = a.mom + (size_t)c * a.P;
  const float *gc = a.grad + (size_t)c * a.P;
  const float eps = a.eps[c];
  const float f = MODE == KICK_FULL_DRIFT ? eps : 0.5f * eps;
  BlockRed v = {3.0e38f, 0.f, 3.0e38f, 0.f, 0.0, 0.0, 0};
  for (int k = blockIdx.y * blockDim.x + threadIdx.x; k < N; k += gridDim.y * blockDim.x) {
    const float p0 = pc[k] + f * gc[k], p1 = pc[N + k] + f * gc[N + k];
    pc[k] = p0;
    pc[N + k] = p1;
    if (MODE == KICK_HALF_LAST) {
      v.s1 += 0.5 * ((double)mi(a, k) * p0 * p0 + (double)mi(a, N + k) * p1 * p1);
      continue;
    }
    const float x0 = xc[k] + eps * mi(a, k) * p0, x1 = xc[N + k] + eps * mi(a, N + k) * p1;
    xc[k] = x0;
    xc[N + k] = x1;
    const NodeH h = node_heights(x0, x1, a.inv_sigma[0], a.inv_sigma[1], a.z_top, false);
    a.H[tix(c, 0, k, N)] = h.H0;
    a.H[tix(c, 1, k, N)] = h.H1;
    a.Hlo[tix(c, 0, k, N)] = h.L0;
    a.Hlo[tix(c, 1, k, N)] = h.L1;
    v.mn0 = fminf(v.mn0, h.H0); v.mx0 = fmaxf(v.mx0, h.H0);
    v.mn1 = fminf(v.mn1, h.H1); v.mx1 = fmaxf(v.mx1, h.H1);
  }
  const BlockRed r = block_reduce(v);
  unsigned *bi = m.bandi + 4 * c;
  if (threadIdx.x == 0) {
    if (MODE == KICK_HALF_LAST) {
      atomicAdd(m.red + 3 * c + 1, r.s1);
    } else {   // non-negative floats order like their bit patterns
      atomicMin(bi + 0, __float_as_uint(r.mn0));
      atomicMax(bi + 1, __float_as_uint(r.mx0));
      atomicMin(bi + 2, __float_as_uint(r.mn1));
      atomicMax(bi + 3, __float_as_uint(r.mx1));
    }
  }
  if (mb_last(m.ticket, c) && threadIdx.x == 0) {
    if (MODE == KICK_HALF_LAST) {
      volatile double *rd = m.red + 3 * c;
      if (a.kin) a.kin[c] = (float)rd[1];
      rd[1] = 0.0;
    } else {
      volatile unsigned *vb = bi;
      a.band[c] = make_float4(__uint_as_float(vb[0]), __uint_as_float(vb[1]), __uint_as_float(vb[2]),
                              __uint_as_float(vb[3]));
      vb[0] = 0x7f7fffffu; vb[1] = 0u; vb[2] = 0x7f7fffffu; vb[3] = 0u;
    }
    m.ticket[c] = 0u;
  }
}

// HMC begin: Philox momenta, kinetic energy, save (x, grad, logp), first
// half kick + drift + heights.
__global__ void __launch_bounds__(MT_THREADS) k_hmc_begin(FinishArgs a, const double *logp,
                                                          float *x0s, float *g0s, double *lp0,
                                                          float *kin0, uint64_t seed,
                                                          uint64_t iter, uint64_t chain_offset) {
  const int c = blockIdx.x, N = a.N, P = a.P;
  float *xc = a.x + (size_t)c * P, *pc = a.mom + (size_t)c * P;
  const float *gc = a.grad + (size_t)c * P;
  const float eps = a.eps[c];
  const int nq = (P + 3) / 4;
  BlockRed v = {3.0e38f, -3.0e38f, 3.0e38f, -3.0e38f, 0.0, 0.0, 0};
  for (int q = threadIdx.x; q < nq; q += blockDim.x) {
    double z[4];
    momenta4(seed, iter, chain_offset + c, q, z);
#pragma unroll
    for (int u = 0; u < 4; u++) {
      int k = 4 * q + u;
      if (k < P) {
        const float m = mi(a, k);
        float pz = a.minv ? (float)(z[u] / sqrt((double)m)) : (float)z[u];
        v.s0 += 0.5 * (double)m * pz * pz;
        float g = gc[k], xv = xc[k];
        x0s[(size_t)c * P + k] = xv;
        g0s[(size_t)c * P + k] = g;
        float ph = pz + 0.5f * eps * g;
        pc[k] = ph;
        xc[k] = xv + eps * m * ph;
      }
    }
  }
  __syncthreads();
  if (a.ncp) {   // non-centred: k_ncp_heights follows
    const BlockRed r = block_reduce(v);
    if (threadIdx.x == 0) {
      kin0[c] = (float)r.s0;
      lp0[c] = logp[c];
    }
    return;
  }
  double is0 = a.inv_sigma[0], is1 = a.inv_sigma[1];
  if (a.sample_r) {   // σ of the drifted ρ (f2)
    const Spec sp = block_spectrum(a.cs, N, xc[2 * N], xc[2 * N + 1], false);
    is0 = sp.inv_sigma[0];
    is1 = sp.inv_sigma[1];
  }
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    NodeH h = node_heights(xc[k], xc[N + k], is0, is1, a.z_top, false);
    a.H[tix(c, 0, k, N)] = h.H0;
    a.H[tix(c, 1, k, N)] = h.H1;
    a.Hlo[tix(c, 0, k, N)] = h.L0;
    a.Hlo[tix(c, 1, k, N)] = h.L1;
    v.mn0 = fminf(v.mn0, h.H0); v.mx0 = fmaxf(v.mx0, h.H0);
    v.mn1 = fminf(v.mn1, h.H1); v.mx1 = fmaxf(v.mx1, h.H1);
  }
  BlockRed r = block_reduce(v);
  if (threadIdx.x == 0) {
    a.band[c] = make_float4(r.mn0, r.mx0, r.mn1, r.mx1);
    kin0[c] = (float)r.s0;
    lp0[c] = logp[c];
  }
}

// HMC end: H = -logp + |p|^2/2, accept iff ln u < -ΔH (u: Philox counter
// (0, chain, iter, 1)), divergence (ΔH > 1000 or non-finite) -> reject.
__global__ void __launch_bounds__(MT_THREADS) k_hmc_end(FinishArgs a, const float *x0s,
                                                        const float *g0s, const double *lp0,
                                                        const float *kin0, const float *kin1,
                                                        uint64_t seed, uint64_t iter,
                                                        uint64_t chain_offset, float *acc_prob,
                                                        int32_t *accepted) {
  __shared__ int s_acc;
  const int c = blockIdx.x, P = a.P;
  if (threadIdx.x == 0) {
    double H0 = -lp0[c] + (double)kin0[c];
    double H1 = -a.logp[c] + (double)kin1[c];
    double dH = H1 - H0;
    uint4 w = philox10(make_uint4(0u, (uint32_t)(chain_offset + c), (uint32_t)iter, 1u),
                       make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
    double u = u01(w.x);
    bool fin = isfinite(dH);
    bool div = !fin || dH > 1000.0;
    bool acc = fin && !div && log(u) < -dH;
    acc_prob[c] = fin ? (float)fmin(1.0, exp(-dH)) : 0.f;
    accepted[c] = acc ? 1 : 0;
    if (a.status) a.status[c] = (acc ? a.status[c] : 0) | (div ? MT_STATUS_DIVERGENT : 0);
    if (!acc) a.logp[c] = lp0[c];
    s_acc = acc;
  }
  __syncthreads();
  if (!s_acc) {
    for (int k = threadIdx.x; k < P; k += blockDim.x) {
      a.x[(size_t)c * P + k] = x0s[(size_t)c * P + k];
      a.grad[(size_t)c * P + k] = g0s[(size_t)c * P + k];
    }
  }
}

__global__ void k_momenta(int C, int P, float *mom, uint64_t seed, uint64_t iter,
                          uint64_t chain_offset, const float *minv) {
  const int nq = (P + 3) / 4;
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)C * nq) return;
  int c = (int)(t / nq), q = (int)(t - (int64_t)c * nq);
  double z[4];
  momenta4(seed, iter, chain_offset + c, q, z);
  for (int m = 0; m < 4; m++)
    if (4 * q + m < P)
      mom[(size_t)c * P + 4 * q + m] = minv ? (float)(z[m] / sqrt((double)minv[4 * q + m])) : (float)z[m];
}

__global__ void k_philox(const uint4 *ctr, uint2 key, uint4 *out, int64_t n, int use_curand) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  out[t] = use_curand ? curand_Philox4x32_10(ctr[t], key) : philox10(ctr[t], key);
}

__global__ void k_ffma(float *out, int iters, float a, float b, long long *cycles) {
  float x[8];
#pragma unroll
  for (int k = 0; k < 8; k++) x[k] = threadIdx.x * 1e-3f + k;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int u = 0; u < 8; u++)
#pragma unroll
      for (int k = 0; k < 8; k++) x[k] = fmaf(x[k], a, b);
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; k++) s += x[k];
  if (s == 1234.5f) out[0] = s;
  if (blockIdx.x == 0 && threadIdx.x == 0) *cycles = t1 - t0;
}

// ---------------------------------------------------------------------------
// sampled-r variants of K1 / K3 / kicks (f2).  The fixed-r kernels above stay
// single-pass; here a leapfrog step needs σ(r) of the DRIFTED ρ before the next
// heights, so the update is split: ρ first (one thread), then the spectrum, then
// the nodes.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void heights_nodes_r(const FinishArgs &a, int c, const float *xc, const Spec &sp) {
  BlockRed v = {3.0e38f, -3.0e38f, 3.0e38f, -3.0e38f, 0.0, 0.0, 0};
  for (int k = threadIdx.x; k < a.N; k += blockDim.x) {
    NodeH h = node_heights(xc[k], xc[a.N + k], sp.inv_sigma[0], sp.inv_sigma[1], a.z_top, false);
    a.H[tix(c, 0, k, a.N)] = h.H0;
    a.H[tix(c, 1, k, a.N)] = h.H1;
    a.Hlo[tix(c, 0, k, a.N)] = h.L0;
    a.Hlo[tix(c, 1, k, a.N)] = h.L1;
    v.mn0 = fminf(v.mn0, h.H0); v.mx0 = fmaxf(v.mx0, h.H0);
    v.mn1 = fminf(v.mn1, h.H1); v.mx1 = fmaxf(v.mx1, h.H1);
  }
  BlockRed r = block_reduce(v);
  if (threadIdx.x == 0) a.band[c] = make_float4(r.mn0, r.mx0, r.mn1, r.mx1);
}

__global__ void __launch_bounds__(MT_THREADS) k_heights_r(FinishArgs a, const float *x) {
  const int c = blockIdx.x;
  const float *xc = x + (size_t)c * a.P;
  const Spec sp = block_spectrum(a.cs, a.N, xc[2 * a.N], xc[2 * a.N + 1], false);
  heights_nodes_r(a, c, xc, sp);
}

template <int MODE>
__global__ void __launch_bounds__(MT_THREADS) k_finish_r(FinishArgs a) {
  extern __shared__ float xs[];  // [P] current state of this chain
  __shared__ float s_new[2];
  const int c = blockIdx.x, N = a.N, ny = a.ny, nx = a.nx;
  float *xc = a.x + (size_t)c * a.P;
  for (int k = threadIdx.x; k < a.P; k += blockDim.x) xs[k] = xc[k];
  __syncthreads();
  const Spec sp = block_spectrum(a.cs, N, xs[2 * N], xs[2 * N + 1], a.prior_on != 0);
  float *Gt = const_cast<float *>(a.G);
  float *gc = a.grad + (size_t)c * a.P;
  float *pc = MODE != FIN_PLAIN ? a.mom + (size_t)c * a.P : nullptr;
  const float eps = MODE != FIN_PLAIN ? a.eps[c] : 0.f;
  // quad_l = x_lᵀQx_l, xAx_l = x_lᵀAx_l, tg_l = Σ t·∂ll/∂x_l (= -∂ll/∂σ_l), kinetic, bad
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    const int i = k / ny, j = k - i * ny;
    const float x0 = xs[k], x1 = xs[N + k];
    const NodeH h = node_heights(x0, x1, sp.inv_sigma[0], sp.inv_sigma[1], a.z_top, true);
    const size_t t0 = tix(c, 0, k, N), t1 = tix(c, 1, k, N);
    const float G0 = Gt[t0], G1 = Gt[t1];
    Gt[t0] = 0.f;
    Gt[t1] = 0.f;
    double gx0 = (double)G0 * h.J0 + (double)G1 * h.J10;
    double gx1 = (double)G1 * h.J11;
    acc[4] += h.t0 * gx0;
    acc[5] += h.t1 * gx1;
    if (a.prior_on) {
      const int ip = (i + 1 == nx ? 0 : i + 1) * ny + j, im = (i == 0 ? nx - 1 : i - 1) * ny + j;
      const int jp = i * ny + (j + 1 == ny ? 0 : j + 1), jm = i * ny + (j == 0 ? ny - 1 : j - 1);
#pragma unroll
      for (int l = 0; l < 2; l++) {
        const float *xl = xs + l * N;
        const double xv = xl[k], nb = (double)xl[ip] + xl[im] + xl[jp] + xl[jm];
        const double Qx = 4.0 * xv - sp.r[l] * nb;
        acc[l] += xv * Qx;
        acc[2 + l] += xv * nb;
        if (l == 0) gx0 -= Qx; else gx1 -= Qx;
      }
    }
    const float g0f = (float)gx0, g1f = (float)gx1;
    gc[k] = g0f;
    gc[N + k] = g1f;
    if (!(isfinite(g0f) && isfinite(g1f))) acc[7] = 1.0;
    if (MODE == FIN_LAST) {
      const float p0 = pc[k] + 0.5f * eps * g0f, p1 = pc[N + k] + 0.5f * eps * g1f;
      pc[k] = p0;
      pc[N + k] = p1;
      acc[6] += 0.5 * ((double)mi(a, k) * p0 * p0 + (double)mi(a, N + k) * p1 * p1);
    }
  }
  block_sum<8>(acc);
  if (threadIdx.x == 0) {
    double lp = a.ll[c];
    float gr[2];
#pragma unroll
    for (int l = 0; l < 2; l++) {
      const double r = sp.r[l], drdrho = r * (1.0 - r);
      double g = drdrho * (-acc[4 + l]) * sp.dsig[l];   // ∂ll/∂σ = -Σ t ∂ll/∂x (∂H/∂σ = -t ∂H/∂x)
      if (a.prior_on) {
        g += drdrho * (0.5 * acc[2 + l] + 0.5 * sp.dld[l]) + 1.0 - 2.0 * r;
        lp += -0.5 * acc[l] + 0.5 * sp.ld[l] - 0.5 * N * log(2.0 * M_PI) + log(r) + log(1.0 - r);
      }
      gr[l] = (float)g;
      gc[2 * N + l] = gr[l];
    }
    a.ll[c] = 0.0;
    a.logp[c] = lp;
    const int bad = acc[7] != 0.0 || !isfinite(lp) || !isfinite(gr[0]) || !isfinite(gr[1]);
    if (a.status) a.status[c] = bad ? MT_STATUS_NONFINITE : 0;
    if (MODE == FIN_LAST) {
      double kin = acc[6];
      for (int l = 0; l < 2; l++) {
        const float pr = pc[2 * N + l] + 0.5f * eps * gr[l];
        pc[2 * N + l] = pr;
        kin += 0.5 * (double)mi(a, 2 * N + l) * pr * pr;
      }
      if (a.kin) a.kin[c] = (float)kin;
    }
    if (MODE == FIN_STEP) {   // close this step's half kick, open the next: p += ε g; ρ += ε p
      for (int l = 0; l < 2; l++) {
        const float pr = pc[2 * N + l] + eps * gr[l];
        pc[2 * N + l] = pr;
        s_new[l] = xs[2 * N + l] + eps * mi(a, 2 * N + l) * pr;
        xc[2 * N + l] = s_new[l];
      }
    }
  }
  if (MODE == FIN_STEP) {
    __syncthreads();
    const Spec sn = block_spectrum(a.cs, N, s_new[0], s_new[1], false);
    BlockRed v = {3.0e38f, -3.0e38f, 3.0e38f, -3.0e38f, 0.0, 0.0, 0};
    for (int k = threadIdx.x; k < N; k += blockDim.x) {
      const float p0 = pc[k] + eps * gc[k], p1 = pc[N + k] + eps * gc[N + k];
      pc[k] = p0;
      pc[N + k] = p1;
      const float xn0 = xs[k] + eps * mi(a, k) * p0, xn1 = xs[N + k] + eps * mi(a, N + k) * p1;
      xc[k] = xn0;
      xc[N + k] = xn1;
      const NodeH hn = node_heights(xn0, xn1, sn.inv_sigma[0], sn.inv_sigma[1], a.z_top, false);
      const size_t t0 = tix(c, 0, k, N), t1 = tix(c, 1, k, N);
      a.H[t0] = hn.H0;
      a.H[t1] = hn.H1;
      a.Hlo[t0] = hn.L0;
      a.Hlo[t1] = hn.L1;
      v.mn0 = fminf(v.mn0, hn.H0); v.mx0 = fmaxf(v.mx0, hn.H0);
      v.mn1 = fminf(v.mn1, hn.H1); v.mx1 = fmaxf(v.mx1, hn.H1);
    }
    BlockRed r = block_reduce(v);
    if (threadIdx.x == 0) a.band[c] = make_float4(r.mn0, r.mx0, r.mn1, r.mx1);
  }
}

template <int MODE>
__global__ void __launch_bounds__(MT_THREADS) k_kick_r(FinishArgs a) {
  __shared__ float s_new[2];
  __shared__ double s_kin;
  const int c = blockIdx.x, N = a.N;
  float *xc = a.x + (size_t)c * a.P, *pc = a.mom + (size_t)c * a.P;
  const float *gc = a.grad + (size_t)c * a.P;
  const float eps = a.eps[c];
  const float f = MODE == KICK_FULL_DRIFT ? eps : 0.5f * eps;
  if (threadIdx.x == 0) {
    double kin = 0.0;
    for (int l = 0; l < 2; l++) {
      const float pr = pc[2 * N + l] + f * gc[2 * N + l];
      pc[2 * N + l] = pr;
      kin += 0.5 * (double)mi(a, 2 * N + l) * pr * pr;
      if (MODE != KICK_HALF_LAST) xc[2 * N + l] += eps * mi(a, 2 * N + l) * pr;
      s_new[l] = xc[2 * N + l];
    }
    s_kin = kin;
  }
  __syncthreads();
  Spec sp{};
  if (MODE != KICK_HALF_LAST) sp = block_spectrum(a.cs, N, s_new[0], s_new[1], false);
  BlockRed v = {3.0e38f, -3.0e38f, 3.0e38f, -3.0e38f, 0.0, 0.0, 0};
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    const float p0 = pc[k] + f * gc[k], p1 = pc[N + k] + f * gc[N + k];
    pc[k] = p0;
    pc[N + k] = p1;
    if (MODE == KICK_HALF_LAST) {
      v.s1 += 0.5 * ((double)mi(a, k) * p0 * p0 + (double)mi(a, N + k) * p1 * p1);
      continue;
    }
    const float x0 = xc[k] + eps * mi(a, k) * p0, x1 = xc[N + k] + eps * mi(a, N + k) * p1;
    xc[k] = x0;
    xc[N + k] = x1;
    const NodeH h = node_heights(x0, x1, sp.inv_sigma[0], sp.inv_sigma[1], a.z_top, false);
    a.H[tix(c, 0, k, N)] = h.H0;
    a.H[tix(c, 1, k, N)] = h.H1;
    a.Hlo[tix(c, 0, k, N)] = h.L0;
    a.Hlo[tix(c, 1, k, N)] = h.L1;
    v.mn0 = fminf(v.mn0, h.H0); v.mx0 = fmaxf(v.mx0, h.H0);
    v.mn1 = fminf(v.mn1, h.H1); v.mx1 = fmaxf(v.mx1, h.H1);
  }
  BlockRed r = block_reduce(v);
  if (threadIdx.x == 0) {
    if (MODE == KICK_HALF_LAST) a.kin[c] = (float)(r.s1 + s_kin);
    else a.band[c] = make_float4(r.mn0, r.mx0, r.mn1, r.mx1);
  }
}

// ---------------------------------------------------------------------------
// Batched NUTS (reading R26): all
// chains advance in lockstep, one leapfrog leaf per step; a chain whose tree
// has stopped (U-turn, divergence or the depth cap) idles.  The per-leaf
// evaluation is the hot path (K1 heights in k_nuts_kick, K2 trace, K3
// finish); these kernels hold the tree bookkeeping of one chain per block:
// edges, subtree/tree proposals, momentum sums, U-turn checkpoints, and the
// Philox-driven directions and multinomial choices (oracle.nuts_step).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double block_dot(const float *a, const float *b, int n) {
  double v[1] = {0.0};
  for (int k = threadIdx.x; k < n; k += blockDim.x) v[0] += (double)a[k] * b[k];
  block_sum<1>(v);
  return v[0];
}

// U-turn(p⁻, p⁺, ρ): p⁻·(ρ - (p⁻+p⁺)/2) <= 0 or p⁺·(ρ - (p⁻+p⁺)/2) <= 0
// generalised U-turn with the velocities p# = M^-1 p at both ends (identity: p)
__device__ __forceinline__ bool block_turning(const float *pl, const float *pr, const float *rho, int n,
                                              const float *minv) {
  double v[2] = {0.0, 0.0};
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const double rs = (double)rho[k] - 0.5 * ((double)pl[k] + pr[k]);
    const double m = minv ? (double)minv[k] : 1.0;
    v[0] += m * (double)pl[k] * rs;
    v[1] += m * (double)pr[k] * rs;
  }
  block_sum<2>(v);
  return v[0] <= 0.0 || v[1] <= 0.0;
}

__device__ __forceinline__ double philox_u(uint64_t seed, uint64_t iter, uint64_t chain, uint32_t stream,
                                           uint32_t q) {
  const uint4 w = philox10(make_uint4(q, (uint32_t)chain, (uint32_t)iter, stream),
                           make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
  return u01(w.x);
}

__device__ __forceinline__ void copyP(float *dst, const float *src, int P) {
  for (int k = threadIdx.x; k < P; k += blockDim.x) dst[k] = src[k];
}

__device__ __forceinline__ double logaddexp(double a, double b) {
  if (a == -INFINITY) return b;
  if (b == -INFINITY) return a;
  const double m = fmax(a, b);
  return m + log1p(exp(-fabs(a - b)));
}

// momenta, H0, edges = current state, ρ = p
__global__ void __launch_bounds__(MT_THREADS) k_nuts_begin(FinishArgs a, NutsArgs n, const float *x,
                                                           const double *logp, const float *grad,
                                                           uint64_t seed, uint64_t iter, uint64_t chain_offset) {
  const int c = blockIdx.x, P = a.P;
  const size_t o = (size_t)c * P;
  const int nq = (P + 3) / 4;
  double v[1] = {0.0};
  for (int q = threadIdx.x; q < nq; q += blockDim.x) {
    double z[4];
    momenta4(seed, iter, chain_offset + c, q, z);
#pragma unroll
    for (int m = 0; m < 4; m++) {
      const int k = 4 * q + m;
      if (k < P) {
        const float mm = mi(a, k);
        const float pz = a.minv ? (float)(z[m] / sqrt((double)mm)) : (float)z[m];
        v[0] += 0.5 * (double)mm * pz * pz;
        n.pL[o + k] = pz;
        n.pR[o + k] = pz;
        n.rho[o + k] = pz;
        n.thL[o + k] = x[o + k];
        n.thR[o + k] = x[o + k];
        n.gL[o + k] = grad[o + k];
        n.gR[o + k] = grad[o + k];
      }
    }
  }
  block_sum<1>(v);
  if (threadIdx.x == 0) {
    NutsChain s{};
    s.H0 = -logp[c] + v[0];
    s.logW = 0.0;
    s.lpL = s.lpR = logp[c];
    s.active = 1;
    n.st[c] = s;
  }
}

// depth j: direction, working state = the edge on that side
__global__ void __launch_bounds__(MT_THREADS) k_nuts_subtree_begin(NutsArgs n, int P, int j, uint64_t seed,
                                                                   uint64_t iter, uint64_t chain_offset) {
  const int c = blockIdx.x;
  __shared__ int s_dir, s_act;
  if (threadIdx.x == 0) {
    NutsChain &s = n.st[c];
    s_act = s.active;
    if (s.active) {
      s.dir = philox_u(seed, iter, chain_offset + c, 2u, (uint32_t)j) >= 0.5 ? 1 : -1;
      s.logWs = -INFINITY;
      s.sub_ok = 1;
    }
    s_dir = s.dir;
  }
  __syncthreads();
  if (!s_act) return;
  const size_t o = (size_t)c * P;
  copyP(n.thw + o, (s_dir > 0 ? n.thR : n.thL) + o, P);
  copyP(n.pw + o, (s_dir > 0 ? n.pR : n.pL) + o, P);
  copyP(n.gw + o, (s_dir > 0 ? n.gR : n.gL) + o, P);
  for (int k = threadIdx.x; k < P; k += blockDim.x) n.rhos[o + k] = 0.f;
}

// first half kick + drift of the working state (signed step v·ε), its heights
__global__ void __launch_bounds__(MT_THREADS) k_nuts_kick(FinishArgs a, NutsArgs n) {
  const int c = blockIdx.x, N = a.N, P = a.P;
  const NutsChain s = n.st[c];
  if (!(s.active && s.sub_ok)) return;
  const size_t o = (size_t)c * P;
  const float e = s.dir * a.eps[c];
  float *th = n.thw + o, *pp = n.pw + o;
  const float *gg = n.gw + o;
  for (int k = threadIdx.x; k < P; k += blockDim.x) {
    const float pk = pp[k] + 0.5f * e * gg[k];
    pp[k] = pk;
    th[k] = th[k] + e * mi(a, k) * pk;
  }
  __syncthreads();
  double is0 = a.inv_sigma[0], is1 = a.inv_sigma[1];
  if (a.sample_r) {
    const Spec sp = block_spectrum(a.cs, N, th[2 * N], th[2 * N + 1], false);
    is0 = sp.inv_sigma[0];
    is1 = sp.inv_sigma[1];
  }
  BlockRed v = {3.0e38f, -3.0e38f, 3.0e38f, -3.0e38f, 0.0, 0.0, 0};
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    const NodeH h = node_heights(th[k], th[N + k], is0, is1, a.z_top, false);
    a.H[tix(c, 0, k, N)] = h.H0;
    a.H[tix(c, 1, k, N)] = h.H1;
    a.Hlo[tix(c, 0, k, N)] = h.L0;
    a.Hlo[tix(c, 1, k, N)] = h.L1;
    v.mn0 = fminf(v.mn0, h.H0); v.mx0 = fmaxf(v.mx0, h.H0);
    v.mn1 = fminf(v.mn1, h.H1); v.mx1 = fmaxf(v.mx1, h.H1);
  }
  BlockRed r = block_reduce(v);
  if (threadIdx.x == 0) a.band[c] = make_float4(r.mn0, r.mx0, r.mn1, r.mx1);
}

// leaf `t` of the subtree (global leaf index = s.n_leaf): second half kick,
// energy, divergence, progressive choice, momentum sum, U-turn checkpoints
__global__ void __launch_bounds__(MT_THREADS) k_nuts_leaf(FinishArgs a, NutsArgs n, int t, uint64_t seed,
                                                          uint64_t iter, uint64_t chain_offset) {
  const int c = blockIdx.x, P = a.P;
  __shared__ NutsChain s;
  __shared__ int s_take, s_turn;
  if (threadIdx.x == 0) s = n.st[c];
  __syncthreads();
  if (!(s.active && s.sub_ok)) return;
  const size_t o = (size_t)c * P;
  const float e = s.dir * a.eps[c];
  float *pp = n.pw + o;
  const float *gg = n.gw + o;
  double v[1] = {0.0};
  for (int k = threadIdx.x; k < P; k += blockDim.x) {
    const float pk = pp[k] + 0.5f * e * gg[k];
    pp[k] = pk;
    v[0] += 0.5 * (double)mi(a, k) * pk * pk;
  }
  block_sum<1>(v);
  if (threadIdx.x == 0) {
    const double lpw = n.lpw_out[c];
    const double dH = (-lpw + v[0]) - s.H0;
    s.acc_sum += isfinite(dH) ? fmin(1.0, exp(-dH)) : 0.0;
    s.n_leaf++;
    s_take = 0;
    if (!isfinite(dH) || dH > 1000.0) {
      s.sub_ok = 0;
      s.diverging = 1;
    } else {
      const double lw = logaddexp(s.logWs, -dH);
      const double u = philox_u(seed, iter, chain_offset + c, 3u, (uint32_t)(s.n_leaf - 1));
      s_take = log(u) < -dH - lw;
      if (s_take) s.lps = lpw;
      s.logWs = lw;
    }
    s.lpw = lpw;
  }
  __syncthreads();
  if (!s.sub_ok) {
    if (threadIdx.x == 0) n.st[c] = s;
    return;
  }
  if (s_take) {
    copyP(n.ths + o, n.thw + o, P);
    copyP(n.gs + o, n.gw + o, P);
  }
  float *rhos = n.rhos + o;
  for (int k = threadIdx.x; k < P; k += blockDim.x) rhos[k] += pp[k];
  __syncthreads();
  // iterative U-turn checks (oracle.leaf_ckpt_idxs)
  const int idx_max = __popc((unsigned)t >> 1), idx_min = idx_max - (__ffs(~t) - 1) + 1;
  const size_t cs = (size_t)a.C * P;   // checkpoint stride
  if ((t & 1) == 0) {
    copyP(n.rck + idx_max * cs + o, pp, P);
    copyP(n.rsck + idx_max * cs + o, rhos, P);
  } else {
    if (threadIdx.x == 0) s_turn = 0;
    __syncthreads();
    float *tmp = n.tmp + o;
    for (int i = idx_max; i >= idx_min; i--) {
      const float *rl = n.rck + i * cs + o, *rsl = n.rsck + i * cs + o;
      for (int k = threadIdx.x; k < P; k += blockDim.x) tmp[k] = rhos[k] - rsl[k] + rl[k];
      __syncthreads();
      if (block_turning(rl, pp, tmp, P, n.minv)) {
        if (threadIdx.x == 0) s_turn = 1;
      }
      __syncthreads();
      if (s_turn) break;
    }
    if (threadIdx.x == 0 && s_turn) s.sub_ok = 0;
  }
  if (threadIdx.x == 0) {
    if (s.sub_ok) atomicOr(n.any_sub, 1);
    n.st[c] = s;
  }
}

// end of depth j: merge a valid subtree (biased progressive choice), move the
// edge, tree U-turn; stop the chain otherwise or at the depth cap
__global__ void __launch_bounds__(MT_THREADS) k_nuts_merge(NutsArgs n, int P, int j, int max_depth, float *x,
                                                           double *logp, float *grad, uint64_t seed,
                                                           uint64_t iter, uint64_t chain_offset) {
  const int c = blockIdx.x;
  __shared__ NutsChain s;
  __shared__ int s_take;
  if (threadIdx.x == 0) s = n.st[c];
  __syncthreads();
  if (!s.active) return;
  const size_t o = (size_t)c * P;
  if (!s.sub_ok) {
    if (threadIdx.x == 0) {
      s.depth = j + 1;
      s.active = 0;
      n.st[c] = s;
    }
    return;
  }
  if (threadIdx.x == 0) {
    const double u = philox_u(seed, iter, chain_offset + c, 4u, (uint32_t)j);
    s_take = log(u) < s.logWs - s.logW;
    if (s_take) logp[c] = s.lps;
    s.logW = logaddexp(s.logW, s.logWs);
    if (s.dir > 0) s.lpR = s.lpw; else s.lpL = s.lpw;
    s.depth = j + 1;
  }
  __syncthreads();
  if (s_take) {
    copyP(x + o, n.ths + o, P);
    copyP(grad + o, n.gs + o, P);
  }
  copyP((s.dir > 0 ? n.thR : n.thL) + o, n.thw + o, P);
  copyP((s.dir > 0 ? n.pR : n.pL) + o, n.pw + o, P);
  copyP((s.dir > 0 ? n.gR : n.gL) + o, n.gw + o, P);
  for (int k = threadIdx.x; k < P; k += blockDim.x) n.rho[o + k] += n.rhos[o + k];
  __syncthreads();
  const bool turn = block_turning(n.pL + o, n.pR + o, n.rho + o, P, n.minv);
  if (threadIdx.x == 0) {
    if (turn || j + 1 >= max_depth) s.active = 0;
    else atomicOr(n.any_active, 1);
    n.st[c] = s;
  }
}

__global__ void k_nuts_end(NutsArgs n, int C, float *accept_stat, int32_t *depth, int32_t *n_leaves,
                           int32_t *status) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const NutsChain s = n.st[c];
  accept_stat[c] = (float)(s.acc_sum / (s.n_leaf > 0 ? s.n_leaf : 1));
  if (depth) depth[c] = s.depth;
  if (n_leaves) n_leaves[c] = s.n_leaf;
  if (status) status[c] = (status[c] & ~MT_STATUS_DIVERGENT) | (s.diverging ? MT_STATUS_DIVERGENT : 0);
}

// ---------------------------------------------------------------------------
// Non-centred CAR prior (reading R13d): state
// (z_0, z_1, ρ_0, ρ_1), x_l = U(r_l) z_l with U = Q(r_l)^{-1/2}, the symmetric
// root of the torus CAR covariance, applied as a circulant by the 2-D DFT:
// U = F⁻¹ diag(λ_ab^{-1/2}) F, dU/dr = F⁻¹ diag(½ c_ab λ_ab^{-3/2}) F,
// λ_ab = 4 - r c_ab.  One block per chain; the DFT is separable (rows, then
// columns), in fp64 (x feeds the heights map, HP2), with the twiddles and all
// intermediates in shared memory: 4N doubles of work space.
// ---------------------------------------------------------------------------
struct Dft {
  double *wre, *wim, *vre, *vim;    // [N] each
  const double *tcx, *tsx, *tcy, *tsy;   // cos / sin (2π k / n) for the two axes
  int nx, ny, N;
};

// y = S(v) for the circulant with eigenvalues s_ab = λ^{-1/2} (mode 0) or
// ½ c λ^{-3/2} (mode 1); v(k) gives input element k (row-major [i][j]); the
// result is left in d.vre (real part).  All threads of the block participate.
template <class In>
__device__ void circ_apply_dft(const Dft &d, const double *cs, double r, int mode, In v) {
  const int nx = d.nx, ny = d.ny, N = d.N;
  for (int q = threadIdx.x; q < N; q += blockDim.x) {        // rows: T[i][b] = Σ_j v e^{-2πi bj/ny}
    const int i = q / ny, b = q - i * ny;
    double re = 0.0, im = 0.0;
    int ph = 0;
    for (int j = 0; j < ny; j++) {
      const double x = v(i * ny + j);
      re += x * d.tcy[ph];
      im -= x * d.tsy[ph];
      ph += b;
      if (ph >= ny) ph -= ny;
    }
    d.wre[q] = re;
    d.wim[q] = im;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < N; q += blockDim.x) {        // columns, scaled: V = s_ab Σ_i T e^{-2πi ai/nx}
    const int a = q / ny, b = q - a * ny;
    double re = 0.0, im = 0.0;
    int ph = 0;
    for (int i = 0; i < nx; i++) {
      const double tr = d.wre[i * ny + b], ti = d.wim[i * ny + b], c = d.tcx[ph], s = d.tsx[ph];
      re += tr * c + ti * s;
      im += ti * c - tr * s;
      ph += a;
      if (ph >= nx) ph -= nx;
    }
    const double cab = cs[q], lam = 4.0 - r * cab;
    const double sc = mode == 0 ? rsqrt(lam) : 0.5 * cab * rsqrt(lam) / lam;
    d.vre[q] = re * sc;
    d.vim[q] = im * sc;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < N; q += blockDim.x) {        // inverse columns
    const int i = q / ny, b = q - i * ny;
    double re = 0.0, im = 0.0;
    int ph = 0;
    for (int a = 0; a < nx; a++) {
      const double vr = d.vre[a * ny + b], vi = d.vim[a * ny + b], c = d.tcx[ph], s = d.tsx[ph];
      re += vr * c - vi * s;
      im += vi * c + vr * s;
      ph += i;
      if (ph >= nx) ph -= nx;
    }
    d.wre[q] = re;
    d.wim[q] = im;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < N; q += blockDim.x) {        // inverse rows, real part / N
    const int i = q / ny, j = q - i * ny;
    double re = 0.0;
    int ph = 0;
    for (int b = 0; b < ny; b++) {
      re += d.wre[i * ny + b] * d.tcy[ph] - d.wim[i * ny + b] * d.tsy[ph];
      ph += j;
      if (ph >= ny) ph -= ny;
    }
    d.vre[q] = re / N;
  }
  __syncthreads();
}

__device__ __forceinline__ int bitrev(int v, int bits) { return (int)(__brev((unsigned)v) >> (32 - bits)); }

// Power-of-two sizes: radix-2 FFTs in place on (vre, vim).  Forward: decimation
// in frequency along rows then columns (natural order in, bit-reversed out);
// the eigenvalue scaling reads c_ab at the bit-reversed frequency; inverse:
// decimation in time (bit-reversed in, natural out).  N log2 N butterflies per
// transform instead of the direct sums' N (n_x + n_y).
template <class In>
__device__ void circ_apply_fft(const Dft &d, const double *cs, double r, int mode, In v) {
  const int nx = d.nx, ny = d.ny, N = d.N, bx = __ffs(nx) - 1, by = __ffs(ny) - 1;
  double *re = d.vre, *im = d.vim;
  for (int q = threadIdx.x; q < N; q += blockDim.x) { re[q] = v(q); im[q] = 0.0; }
  __syncthreads();
  // forward DIF along rows (length ny, stride 1) then columns (length nx, stride ny)
  for (int pass = 0; pass < 2; pass++) {
    const int n = pass ? nx : ny, ln = pass ? bx : by, st = pass ? ny : 1, lines = pass ? ny : nx;
    const double *tc = pass ? d.tcx : d.tcy, *ts = pass ? d.tsx : d.tsy;
    for (int lh = ln - 1; lh >= 0; lh--) {
      const int h = 1 << lh, tstep = n >> (lh + 1);
      for (int t = threadIdx.x; t < lines << (ln - 1); t += blockDim.x) {
        // rows: consecutive threads take consecutive butterflies of a row; columns:
        // consecutive columns (a column-major walk would put a warp on one bank)
        const int line = pass ? (t & (lines - 1)) : t >> (ln - 1);
        const int bfly = pass ? t >> by : t & ((n >> 1) - 1);
        const int g = (bfly >> lh) << (lh + 1), k = bfly & (h - 1);
        const int base = pass ? line : line * ny;
        const int i0 = base + (g + k) * st, i1 = i0 + h * st;
        const double ar = re[i0], ai = im[i0], br = re[i1], bi = im[i1];
        const double dr = ar - br, di = ai - bi, c = tc[k * tstep], sn = ts[k * tstep];
        re[i0] = ar + br;
        im[i0] = ai + bi;
        re[i1] = dr * c + di * sn;      // (a - b) e^{-iθ}
        im[i1] = di * c - dr * sn;
      }
      __syncthreads();
    }
  }
  for (int q = threadIdx.x; q < N; q += blockDim.x) {        // eigenvalues at bit-reversed frequencies
    const int pi = q >> by, pj = q & (ny - 1);
    const double cab = cs[bitrev(pi, bx) * ny + bitrev(pj, by)], lam = 4.0 - r * cab;
    const double sc = (mode == 0 ? rsqrt(lam) : 0.5 * cab * rsqrt(lam) / lam) / N;
    re[q] *= sc;
    im[q] *= sc;
  }
  __syncthreads();
  // inverse DIT along columns then rows
  for (int pass = 0; pass < 2; pass++) {
    const int n = pass ? ny : nx, ln = pass ? by : bx, st = pass ? 1 : ny, lines = pass ? nx : ny;
    const double *tc = pass ? d.tcy : d.tcx, *ts = pass ? d.tsy : d.tsx;
    for (int lh = 0; lh < ln; lh++) {
      const int h = 1 << lh, tstep = n >> (lh + 1);
      for (int t = threadIdx.x; t < lines << (ln - 1); t += blockDim.x) {
        const int line = pass ? t >> (ln - 1) : (t & (lines - 1));   // pass 0: columns
        const int bfly = pass ? t & ((n >> 1) - 1) : t >> by;
        const int g = (bfly >> lh) << (lh + 1), k = bfly & (h - 1);
        const int base = pass ? line * ny : line;
        const int i0 = base + (g + k) * st, i1 = i0 + h * st;
        const double c = tc[k * tstep], sn = ts[k * tstep];
        const double br = re[i1] * c - im[i1] * sn, bi = im[i1] * c + re[i1] * sn;   // b e^{+iθ}
        const double ar = re[i0], ai = im[i0];
        re[i0] = ar + br;
        im[i0] = ai + bi;
        re[i1] = ar - br;
        im[i1] = ai - bi;
      }
      __syncthreads();
    }
  }
}

#ifndef MT_FFT_MIN_N
#define MT_FFT_MIN_N 0
#endif
template <class In>
__device__ __forceinline__ void circ_apply(const Dft &d, const double *cs, double r, int mode, In v) {
  // power-of-two grids: FFT (measured per evaluation, Medium n = 32: DFT 6.01 vs FFT 5.61 ms;
  // ray-sharded n = 64: DFT 1.50 vs FFT 0.71 ms); other sizes: the direct sums
  if ((d.nx & (d.nx - 1)) == 0 && (d.ny & (d.ny - 1)) == 0 && d.N >= MT_FFT_MIN_N) circ_apply_fft(d, cs, r, mode, v);
  else circ_apply_dft(d, cs, r, mode, v);
}

__device__ __forceinline__ Dft dft_setup(double *sm, int nx, int ny) {
  Dft d;
  d.nx = nx; d.ny = ny; d.N = nx * ny;
  d.wre = sm; d.wim = sm + d.N; d.vre = sm + 2 * d.N; d.vim = sm + 3 * d.N;
  double *tw = sm + 4 * d.N;
  for (int k = threadIdx.x; k < nx; k += blockDim.x) {
    double sn, c;
    sincospi(2.0 * k / nx, &sn, &c);
    tw[k] = c;
    tw[MT_MAX_AXIS + k] = sn;
  }
  for (int k = threadIdx.x; k < ny; k += blockDim.x) {
    double sn, c;
    sincospi(2.0 * k / ny, &sn, &c);
    tw[2 * MT_MAX_AXIS + k] = c;
    tw[3 * MT_MAX_AXIS + k] = sn;
  }
  d.tcx = tw; d.tsx = tw + MT_MAX_AXIS; d.tcy = tw + 2 * MT_MAX_AXIS; d.tsy = tw + 3 * MT_MAX_AXIS;
  __syncthreads();
  return d;
}

// K1 (non-centred): x_l = U(r_l) z_l (fp64, kept in a.xw for K3), heights, band.
__global__ void __launch_bounds__(MT_THREADS) k_ncp_heights(FinishArgs a, const float *v) {
  extern __shared__ double sm[];
  const int c = blockIdx.x, N = a.N;
  const float *vc = v + (size_t)c * a.P;
  const Spec sp = block_spectrum(a.cs, N, vc[2 * N], vc[2 * N + 1], false);
  const Dft d = dft_setup(sm, a.nx, a.ny);
  double *xw = a.xw + (size_t)c * 2 * N;
  for (int l = 0; l < 2; l++) {
    const float *z = vc + l * N;
    circ_apply(d, a.cs, sp.r[l], 0, [&](int k) { return (double)z[k]; });
    for (int k = threadIdx.x; k < N; k += blockDim.x) xw[l * N + k] = d.vre[k];
    __syncthreads();
  }
  BlockRed vr = {3.0e38f, -3.0e38f, 3.0e38f, -3.0e38f, 0.0, 0.0, 0};
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    const NodeH h = node_heights(xw[k], xw[N + k], sp.inv_sigma[0], sp.inv_sigma[1], a.z_top, false);
    a.H[tix(c, 0, k, N)] = h.H0;
    a.H[tix(c, 1, k, N)] = h.H1;
    a.Hlo[tix(c, 0, k, N)] = h.L0;
    a.Hlo[tix(c, 1, k, N)] = h.L1;
    vr.mn0 = fminf(vr.mn0, h.H0); vr.mx0 = fmaxf(vr.mx0, h.H0);
    vr.mn1 = fminf(vr.mn1, h.H1); vr.mx1 = fmaxf(vr.mx1, h.H1);
  }
  const BlockRed r = block_reduce(vr);
  if (threadIdx.x == 0) a.band[c] = make_float4(r.mn0, r.mx0, r.mn1, r.mx1);
}

// K3 (non-centred): ∂ll/∂x from ∂ll/∂H, then
//   ∂/∂z_l = -z_l + U ∂ll/∂x_l,  ∂/∂ρ_l = r(1-r)[(∂ll/∂x_l)ᵀ (dU/dr) z_l + (∂ll/∂σ_l) dσ_l/dr] + 1 - 2r,
//   logp = ll - ½|z|² - N ln 2π + Σ_l ln r_l(1 - r_l)   (prior terms on the prior-owning shard).
__global__ void __launch_bounds__(MT_THREADS) k_ncp_finish(FinishArgs a) {
  extern __shared__ double sm[];
  const int c = blockIdx.x, N = a.N, P = a.P;
  const float *vc = a.x + (size_t)c * P;
  float *gc = a.grad + (size_t)c * P;
  const Spec sp = block_spectrum(a.cs, N, vc[2 * N], vc[2 * N + 1], false);
  double *gx = sm + 4 * N + 4 * MT_MAX_AXIS;   // [2N] ∂ll/∂x
  const double *xw = a.xw + (size_t)c * 2 * N;
  float *Gt = const_cast<float *>(a.G);
  double acc[4] = {0.0, 0.0, 0.0, 0.0};   // Σ t0 gx0, Σ t1 gx1, Σ z², bad
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    const NodeH h = node_heights(xw[k], xw[N + k], sp.inv_sigma[0], sp.inv_sigma[1], a.z_top, true);
    const size_t t0 = tix(c, 0, k, N), t1 = tix(c, 1, k, N);
    const double G0 = Gt[t0], G1 = Gt[t1];
    Gt[t0] = 0.f;
    Gt[t1] = 0.f;
    const double gx0 = G0 * h.J0 + G1 * h.J10, gx1 = G1 * h.J11;
    gx[k] = gx0;
    gx[N + k] = gx1;
    acc[0] += h.t0 * gx0;
    acc[1] += h.t1 * gx1;
    const double z0 = vc[k], z1 = vc[N + k];
    acc[2] += z0 * z0 + z1 * z1;
  }
  block_sum<4>(acc);
  const Dft d = dft_setup(sm, a.nx, a.ny);
  double gr[2];
  int bad = 0;
  for (int l = 0; l < 2; l++) {
    const double *g = gx + l * N;
    circ_apply(d, a.cs, sp.r[l], 0, [&](int k) { return g[k]; });   // U ∂ll/∂x_l
    for (int k = threadIdx.x; k < N; k += blockDim.x) {
      const float gz = (float)((a.prior_on ? -(double)vc[l * N + k] : 0.0) + d.vre[k]);
      gc[l * N + k] = gz;
      bad |= !isfinite(gz);
    }
    __syncthreads();
    const float *z = vc + l * N;
    circ_apply(d, a.cs, sp.r[l], 1, [&](int k) { return (double)z[k]; });   // (dU/dr) z_l
    double s[1] = {0.0};
    for (int k = threadIdx.x; k < N; k += blockDim.x) s[0] += g[k] * d.vre[k];
    block_sum<1>(s);
    const double r = sp.r[l];
    // ∂ll/∂σ_l = Σ ∂ll/∂H ∂H/∂σ = -Σ t_l ∂ll/∂x_l  (t = x/σ inside the clamp)
    const double dll_ds = -acc[l];
    gr[l] = r * (1.0 - r) * (s[0] + dll_ds * sp.dsig[l]) + (a.prior_on ? 1.0 - 2.0 * r : 0.0);
  }
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) {
    gc[2 * N] = (float)gr[0];
    gc[2 * N + 1] = (float)gr[1];
    double lp = a.ll[c];
    if (a.prior_on)
      lp += -0.5 * acc[2] - N * log(2.0 * M_PI) + log(sp.r[0]) + log1p(-sp.r[0]) + log(sp.r[1]) + log1p(-sp.r[1]);
    a.ll[c] = 0.0;
    a.logp[c] = lp;
    if (a.status) a.status[c] = (bad || !isfinite(lp) || !isfinite(gr[0]) || !isfinite(gr[1])) ? MT_STATUS_NONFINITE : 0;
  }
}

// Cluster variants: a 2-CTA thread-block cluster per chain, CTA l = surface l,
// so a chain's two surfaces transform on two SMs at once.  The heights need
// x_0 and x_1 at every node: each CTA reads its partner's x through
// distributed shared memory; the per-chain scalars meet the same way.
namespace cgx = cooperative_groups;

__global__ void __cluster_dims__(1, 2, 1) __launch_bounds__(MT_THREADS) k_ncp_heights_cl(FinishArgs a, const float *v) {
  extern __shared__ double sm[];
  cgx::cluster_group cluster = cgx::this_cluster();
  const int c = blockIdx.x, l = blockIdx.y, N = a.N;
  const float *vc = v + (size_t)c * a.P;
  const Spec sp = block_spectrum(a.cs, N, vc[2 * N], vc[2 * N + 1], false);
  const Dft d = dft_setup(sm, a.nx, a.ny);
  double *xl = sm + 4 * N + 4 * MT_MAX_AXIS;   // [N] this surface's x
  __shared__ float bandp[4];
  const float *z = vc + l * N;
  circ_apply(d, a.cs, sp.r[l], 0, [&](int k) { return (double)z[k]; });
  double *xw = a.xw + (size_t)c * 2 * N + (size_t)l * N;
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    xl[k] = d.vre[k];
    xw[k] = d.vre[k];
  }
  cluster.sync();
  const double *x0 = l == 0 ? xl : cluster.map_shared_rank(xl, 0);
  const double *x1 = l == 1 ? xl : cluster.map_shared_rank(xl, 1);
  BlockRed vr = {3.0e38f, -3.0e38f, 3.0e38f, -3.0e38f, 0.0, 0.0, 0};
  const int half = (N + 1) / 2, k0 = l * half, k1 = min(N, k0 + half);   // CTA l: half of the nodes
  for (int k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
    const NodeH h = node_heights(x0[k], x1[k], sp.inv_sigma[0], sp.inv_sigma[1], a.z_top, false);
    a.H[tix(c, 0, k, N)] = h.H0;
    a.H[tix(c, 1, k, N)] = h.H1;
    a.Hlo[tix(c, 0, k, N)] = h.L0;
    a.Hlo[tix(c, 1, k, N)] = h.L1;
    vr.mn0 = fminf(vr.mn0, h.H0); vr.mx0 = fmaxf(vr.mx0, h.H0);
    vr.mn1 = fminf(vr.mn1, h.H1); vr.mx1 = fmaxf(vr.mx1, h.H1);
  }
  const BlockRed r = block_reduce(vr);
  if (threadIdx.x == 0) { bandp[0] = r.mn0; bandp[1] = r.mx0; bandp[2] = r.mn1; bandp[3] = r.mx1; }
  cluster.sync();
  if (l == 0 && threadIdx.x == 0) {
    const float *o = cluster.map_shared_rank(bandp, 1);
    a.band[c] = make_float4(fminf(bandp[0], o[0]), fmaxf(bandp[1], o[1]), fminf(bandp[2], o[2]), fmaxf(bandp[3], o[3]));
  }
  cluster.sync();   // keep this CTA's shared memory alive until the partner has read it
}

__global__ void __cluster_dims__(1, 2, 1) __launch_bounds__(MT_THREADS) k_ncp_finish_cl(FinishArgs a) {
  extern __shared__ double sm[];
  cgx::cluster_group cluster = cgx::this_cluster();
  const int c = blockIdx.x, l = blockIdx.y, N = a.N, P = a.P;
  const float *vc = a.x + (size_t)c * P;
  float *gc = a.grad + (size_t)c * P;
  const Spec sp = block_spectrum(a.cs, N, vc[2 * N], vc[2 * N + 1], false);
  double *gx = sm + 4 * N + 4 * MT_MAX_AXIS;   // [N] ∂ll/∂x_l
  __shared__ double part[3];                   // Σ z_l², non-finite flag, ∂/∂ρ_l
  const double *xw = a.xw + (size_t)c * 2 * N;
  const float *Gt = a.G;
  double acc[2] = {0.0, 0.0};   // Σ t_l gx_l, Σ z_l²
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    const NodeH h = node_heights(xw[k], xw[N + k], sp.inv_sigma[0], sp.inv_sigma[1], a.z_top, true);
    const double G0 = Gt[tix(c, 0, k, N)], G1 = Gt[tix(c, 1, k, N)];
    const double g = l == 0 ? G0 * h.J0 + G1 * h.J10 : G1 * h.J11;
    gx[k] = g;
    acc[0] += (l == 0 ? h.t0 : h.t1) * g;
    const double zv = vc[l * N + k];
    acc[1] += zv * zv;
  }
  block_sum<2>(acc);
  cluster.sync();   // both CTAs have read ∂ℓ/∂H: clear it (CTA l its surface)
  float *Gw = const_cast<float *>(a.G);
  for (int k = threadIdx.x; k < N; k += blockDim.x) Gw[tix(c, l, k, N)] = 0.f;
  const Dft d = dft_setup(sm, a.nx, a.ny);
  int bad = 0;
  circ_apply(d, a.cs, sp.r[l], 0, [&](int k) { return gx[k]; });   // U ∂ll/∂x_l
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    const float gz = (float)((a.prior_on ? -(double)vc[l * N + k] : 0.0) + d.vre[k]);
    gc[l * N + k] = gz;
    bad |= !isfinite(gz);
  }
  __syncthreads();
  const float *z = vc + l * N;
  circ_apply(d, a.cs, sp.r[l], 1, [&](int k) { return (double)z[k]; });   // (dU/dr) z_l
  double sdot[1] = {0.0};
  for (int k = threadIdx.x; k < N; k += blockDim.x) sdot[0] += gx[k] * d.vre[k];
  block_sum<1>(sdot);
  bad = __syncthreads_or(bad);
  const double r = sp.r[l];
  const double gr = r * (1.0 - r) * (sdot[0] - acc[0] * sp.dsig[l]) + (a.prior_on ? 1.0 - 2.0 * r : 0.0);
  if (threadIdx.x == 0) {
    gc[2 * N + l] = (float)gr;
    part[0] = acc[1];
    part[1] = (bad || !isfinite(gr)) ? 1.0 : 0.0;
  }
  cluster.sync();
  if (l == 0 && threadIdx.x == 0) {
    const double *o = cluster.map_shared_rank(part, 1);
    double lp = a.ll[c];
    if (a.prior_on)
      lp += -0.5 * (part[0] + o[0]) - N * log(2.0 * M_PI) + log(sp.r[0]) + log1p(-sp.r[0]) + log(sp.r[1]) +
            log1p(-sp.r[1]);
    a.ll[c] = 0.0;
    a.logp[c] = lp;
    if (a.status) a.status[c] = (part[1] != 0.0 || o[1] != 0.0 || !isfinite(lp)) ? MT_STATUS_NONFINITE : 0;
  }
  cluster.sync();
}

// Leapfrog kicks / drifts in the non-centred coordinates (heights follow in
// k_ncp_heights): KICK_HALF_DRIFT p += ε/2 g, z += ε p; KICK_FULL_DRIFT p += ε g,
// z += ε p; KICK_HALF_LAST p += ε/2 g and the kinetic energy ½|p|².
template <int MODE>
__global__ void __launch_bounds__(MT_THREADS) k_ncp_kick(FinishArgs a) {
  const int c = blockIdx.x, P = a.P;
  float *xc = a.x + (size_t)c * P, *pc = a.mom + (size_t)c * P;
  const float *gc = a.grad + (size_t)c * P;
  const float eps = a.eps[c], f = MODE == KICK_FULL_DRIFT ? eps : 0.5f * eps;
  double kin[1] = {0.0};
  for (int k = threadIdx.x; k < P; k += blockDim.x) {
    const float p = pc[k] + f * gc[k];
    pc[k] = p;
    if (MODE != KICK_HALF_LAST) xc[k] = xc[k] + eps * mi(a, k) * p;
    else kin[0] += 0.5 * (double)mi(a, k) * p * p;
  }
  if (MODE == KICK_HALF_LAST) {
    block_sum<1>(kin);
    if (threadIdx.x == 0 && a.kin) a.kin[c] = (float)kin[0];
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
// few-chain multi-block K3 / kicks (fixed r, centred): blocks per chain so that
// about 2 blocks per SM are in flight
bool use_mb(const mt_problem *p, int C) {
  return p->mb_red != nullptr && C < 16 && !p->sample_r && !p->ncp;
}
static int mb_blocks(const mt_problem *p, int C) {
  int nb = (2 * p->num_sms + C - 1) / C;
  const int cap = (p->N + MT_THREADS - 1) / MT_THREADS;
  return nb < 1 ? 1 : (nb > cap ? cap : nb);
}
static MbScratch mb_scratch(mt_problem *p) {
  MbScratch m;
  m.red = p->mb_red;
  m.bandi = p->mb_band;
  m.ticket = p->mb_ticket;
  return m;
}

// dynamic shared memory of the non-centred kernels: 4N doubles of DFT work + twiddles
// (K3 adds 2N for ∂ll/∂x): up to 200 KiB at N = 4096, so opt in once
static size_t ncp_smem(const mt_problem *p) {
  static bool attr = false;
  if (!attr) {
    const int mx = (6 * MT_MAX_NODES + 4 * MT_MAX_AXIS) * (int)sizeof(double);
    cudaFuncSetAttribute(k_ncp_heights, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(k_ncp_finish, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(k_ncp_heights_cl, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(k_ncp_finish_cl, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    attr = true;
  }
  return (size_t)(4 * p->N + 4 * MT_MAX_AXIS) * sizeof(double);
}

#ifndef MT_NCP_CLUSTER
#define MT_NCP_CLUSTER 1
#endif
static void launch_ncp_heights(mt_problem *p, const FinishArgs &a, int C, const float *x, cudaStream_t s) {
  if (MT_NCP_CLUSTER)
    k_ncp_heights_cl<<<dim3(C, 2), MT_THREADS, ncp_smem(p) + (size_t)p->N * sizeof(double), s>>>(a, x);
  else
    k_ncp_heights<<<C, MT_THREADS, ncp_smem(p), s>>>(a, x);
}

static FinishArgs base_args(mt_problem *p, int C) {
  FinishArgs a{};
  a.nx = p->nx; a.ny = p->ny; a.N = p->N; a.P = p->P; a.C = C;
  a.z_top = p->z_top;
  a.inv_sigma[0] = 1.0 / p->sigma[0];
  a.inv_sigma[1] = 1.0 / p->sigma[1];
  a.car_r[0] = p->car_r[0];
  a.car_r[1] = p->car_r[1];
  a.prior_const = 0.0;
  for (int l = 0; l < 2; l++) a.prior_const += 0.5 * p->logdetQ[l] - 0.5 * p->N * log(2.0 * M_PI);
  a.prior_on = p->prior_on;
  a.G = p->d_G;
  a.ll = p->d_ll;
  a.H = p->d_H;
  a.Hlo = p->d_Hlo;
  a.band = p->d_band;
  a.sample_r = p->sample_r;
  a.cs = p->d_cs;
  a.ncp = p->ncp;
  a.xw = p->d_xw;
  a.minv = p->d_minv;
  return a;
}

cudaError_t launch_heights(mt_problem *p, int C, const float *x, float *H, float4 *band,
                           cudaStream_t s) {
  if (C <= 0) return cudaSuccess;
  FinishArgs a = base_args(p, C);
  a.H = H;
  a.Hlo = p->d_Hlo;
  a.band = band;
  if (p->ncp) launch_ncp_heights(p, a, C, x, s);
  else if (p->sample_r) k_heights_r<<<C, MT_THREADS, 0, s>>>(a, x);
  else k_heights<<<C, MT_THREADS, 0, s>>>(a, x);
  p->all_launches++;
  return cudaGetLastError();
}

cudaError_t launch_finish(mt_problem *p, int mode, int C, float *x, float *grad, double *logp,
                          int32_t *status, float *mom, const float *eps, float *kin,
                          cudaStream_t s) {
  if (C <= 0) return cudaSuccess;
  FinishArgs a = base_args(p, C);
  a.x = x; a.grad = grad; a.logp = logp; a.status = status; a.mom = mom; a.eps = eps; a.kin = kin;
  if (use_mb(p, C)) {   // few chains: several blocks per chain (unfused leapfrog)
    if (mode != FIN_PLAIN) return cudaErrorInvalidValue;
    k_finish_mb<<<dim3(C, mb_blocks(p, C)), MT_THREADS, 0, s>>>(a, mb_scratch(p));
    p->all_launches++;
    return cudaGetLastError();
  }
  if (p->ncp) {   // unfused: the API drives kicks / drifts separately (k_ncp_kick)
    if (mode != FIN_PLAIN) return cudaErrorInvalidValue;
    if (MT_NCP_CLUSTER)
      k_ncp_finish_cl<<<dim3(C, 2), MT_THREADS, ncp_smem(p) + (size_t)p->N * sizeof(double), s>>>(a);
    else
      k_ncp_finish<<<C, MT_THREADS, ncp_smem(p) + (size_t)2 * p->N * sizeof(double), s>>>(a);
    p->all_launches++;
    return cudaGetLastError();
  }
  size_t smem = (size_t)p->P * sizeof(float);
  static bool attr[3] = {false, false, false};
  if (smem > 48 * 1024 && !attr[mode]) {
    if (mode == FIN_PLAIN)
      cudaFuncSetAttribute(k_finish<FIN_PLAIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    if (mode == FIN_STEP)
      cudaFuncSetAttribute(k_finish<FIN_STEP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    if (mode == FIN_LAST)
      cudaFuncSetAttribute(k_finish<FIN_LAST>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    attr[mode] = true;
  }
  if (p->sample_r) {
    static bool attr_r[3] = {false, false, false};
    if (smem > 48 * 1024 && !attr_r[mode]) {
      if (mode == FIN_PLAIN)
        cudaFuncSetAttribute(k_finish_r<FIN_PLAIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
      if (mode == FIN_STEP)
        cudaFuncSetAttribute(k_finish_r<FIN_STEP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
      if (mode == FIN_LAST)
        cudaFuncSetAttribute(k_finish_r<FIN_LAST>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
      attr_r[mode] = true;
    }
    if (mode == FIN_PLAIN) k_finish_r<FIN_PLAIN><<<C, MT_THREADS, smem, s>>>(a);
    else if (mode == FIN_STEP) k_finish_r<FIN_STEP><<<C, MT_THREADS, smem, s>>>(a);
    else k_finish_r<FIN_LAST><<<C, MT_THREADS, smem, s>>>(a);
  } else if (mode == FIN_PLAIN) k_finish<FIN_PLAIN><<<C, MT_THREADS, smem, s>>>(a);
  else if (mode == FIN_STEP) k_finish<FIN_STEP><<<C, MT_THREADS, smem, s>>>(a);
  else k_finish<FIN_LAST><<<C, MT_THREADS, smem, s>>>(a);
  p->all_launches++;
  return cudaGetLastError();
}

cudaError_t launch_kick(mt_problem *p, int mode, int C, float *x, float *mom, const float *grad,
                        const float *eps, float *kin, cudaStream_t s) {
  if (C <= 0) return cudaSuccess;
  FinishArgs a = base_args(p, C);
  a.x = x; a.mom = mom; a.grad = const_cast<float *>(grad); a.eps = eps; a.kin = kin;
  if (use_mb(p, C)) {
    const dim3 g(C, mb_blocks(p, C));
    if (mode == KICK_HALF_DRIFT) k_kick_mb<KICK_HALF_DRIFT><<<g, MT_THREADS, 0, s>>>(a, mb_scratch(p));
    else if (mode == KICK_FULL_DRIFT) k_kick_mb<KICK_FULL_DRIFT><<<g, MT_THREADS, 0, s>>>(a, mb_scratch(p));
    else k_kick_mb<KICK_HALF_LAST><<<g, MT_THREADS, 0, s>>>(a, mb_scratch(p));
    p->all_launches++;
    return cudaGetLastError();
  }
  if (p->ncp) {
    if (mode == KICK_HALF_DRIFT) k_ncp_kick<KICK_HALF_DRIFT><<<C, MT_THREADS, 0, s>>>(a);
    else if (mode == KICK_FULL_DRIFT) k_ncp_kick<KICK_FULL_DRIFT><<<C, MT_THREADS, 0, s>>>(a);
    else k_ncp_kick<KICK_HALF_LAST><<<C, MT_THREADS, 0, s>>>(a);
    p->all_launches++;
    if (mode != KICK_HALF_LAST) {
      launch_ncp_heights(p, a, C, x, s);
      p->all_launches++;
    }
    return cudaGetLastError();
  }
  if (p->sample_r) {
    if (mode == KICK_HALF_DRIFT) k_kick_r<KICK_HALF_DRIFT><<<C, MT_THREADS, 0, s>>>(a);
    else if (mode == KICK_FULL_DRIFT) k_kick_r<KICK_FULL_DRIFT><<<C, MT_THREADS, 0, s>>>(a);
    else k_kick_r<KICK_HALF_LAST><<<C, MT_THREADS, 0, s>>>(a);
  } else if (mode == KICK_HALF_DRIFT) k_kick<KICK_HALF_DRIFT><<<C, MT_THREADS, 0, s>>>(a);
  else if (mode == KICK_FULL_DRIFT) k_kick<KICK_FULL_DRIFT><<<C, MT_THREADS, 0, s>>>(a);
  else k_kick<KICK_HALF_LAST><<<C, MT_THREADS, 0, s>>>(a);
  p->all_launches++;
  return cudaGetLastError();
}

cudaError_t launch_kick_drift(mt_problem *p, int C, float *x, float *mom, const float *grad,
                              const float *eps, cudaStream_t s) {
  return launch_kick(p, KICK_HALF_DRIFT, C, x, mom, grad, eps, nullptr, s);
}

cudaError_t launch_hmc_begin(mt_problem *p, int C, float *x, const double *logp,
                             const float *grad, const float *eps, uint64_t seed, uint64_t iter,
                             uint64_t chain_offset, cudaStream_t s) {
  FinishArgs a = base_args(p, C);
  a.x = x; a.mom = p->d_mom; a.grad = const_cast<float *>(grad); a.eps = eps;
  k_hmc_begin<<<C, MT_THREADS, 0, s>>>(a, logp, p->d_x0, p->d_g0, p->d_lp0, p->d_kin0, seed, iter,
                                       chain_offset);
  p->all_launches++;
  if (p->ncp) {   // heights of the drifted z (k_hmc_begin skipped them)
    launch_ncp_heights(p, a, C, x, s);
    p->all_launches++;
  }
  return cudaGetLastError();
}

cudaError_t launch_hmc_end(mt_problem *p, int C, float *x, double *logp, float *grad,
                           uint64_t seed, uint64_t iter, uint64_t chain_offset, float *acc_prob,
                           int32_t *accepted, int32_t *status, cudaStream_t s) {
  FinishArgs a = base_args(p, C);
  a.x = x; a.logp = logp; a.grad = grad; a.status = status;
  k_hmc_end<<<C, MT_THREADS, 0, s>>>(a, p->d_x0, p->d_g0, p->d_lp0, p->d_kin0, p->d_kin1, seed,
                                     iter, chain_offset, acc_prob, accepted);
  p->all_launches++;
  return cudaGetLastError();
}

cudaError_t launch_momenta(mt_problem *p, int C, float *mom, uint64_t seed, uint64_t iter,
                           uint64_t chain_offset, cudaStream_t s) {
  if (C <= 0) return cudaSuccess;
  int64_t n = (int64_t)C * ((p->P + 3) / 4);
  k_momenta<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(C, p->P, mom, seed, iter, chain_offset, p->d_minv);
  p->all_launches++;
  return cudaGetLastError();
}

cudaError_t launch_philox(const uint32_t *ctr, uint32_t k0, uint32_t k1, uint32_t *out, int64_t n,
                          int use_curand, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  k_philox<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(reinterpret_cast<const uint4 *>(ctr),
                                                       make_uint2(k0, k1),
                                                       reinterpret_cast<uint4 *>(out), n, use_curand);
  return cudaGetLastError();
}

// [C][2][N] <-> chain-interleaved [C/32][2][N][32]
__global__ void k_tile(int C, int N, const float *src, float *dst, int to_tiled) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)C * 2 * N) return;
  int c = (int)(t / (2 * N)), m = (int)(t - (int64_t)c * 2 * N);
  size_t ti = tix(c, m / N, m % N, N);
  if (to_tiled) dst[ti] = src[t];
  else dst[t] = src[ti];
}

cudaError_t launch_tile(mt_problem *p, int C, const float *src, float *dst, int to_tiled,
                        cudaStream_t s) {
  if (C <= 0) return cudaSuccess;
  int64_t n = (int64_t)C * 2 * p->N;
  k_tile<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(C, p->N, src, dst, to_tiled);
  p->all_launches++;
  return cudaGetLastError();
}

cudaError_t run_fp32_peak(int device, double *tflops, double *mhz) {
  cudaDeviceProp prop;
  cudaError_t e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) return e;
  float *out;
  long long *cyc;
  cudaMalloc(&out, sizeof(float));
  cudaMalloc(&cyc, sizeof(long long));
  int blocks = prop.multiProcessorCount * 4, threads = 512, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_ffma<<<blocks, threads>>>(out, 64, 1.0000001f, 1e-7f, cyc);  // warm-up
  double best = 0, best_mhz = 0;
  for (int rep = 0; rep < 10; rep++) {
    cudaEventRecord(e0);
    k_ffma<<<blocks, threads>>>(out, iters, 1.0000001f, 1e-7f, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    long long cycles = 0;
    cudaMemcpy(&cycles, cyc, sizeof(long long), cudaMemcpyDeviceToHost);
    double fl = 2.0 * 64.0 * iters * (double)blocks * threads;
    double tf = fl / (ms * 1e-3) / 1e12;
    if (tf > best) { best = tf; best_mhz = cycles / (ms * 1e3); }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  cudaFree(cyc);
  *tflops = best;
  *mhz = best_mhz;
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// NUTS transition (host loop over depths and leaves; see k_nuts_*)
// ---------------------------------------------------------------------------
static cudaError_t nuts_workspace(mt_problem *p) {
  if (p->nuts_ws) return cudaSuccess;
  const size_t CP = (size_t)(p->max_chains > 0 ? p->max_chains : 1) * p->P;
  const size_t nf = CP * (16 + 2 * MT_NUTS_MAX_DEPTH);
  cudaError_t e = cudaMalloc(&p->nuts_ws, sizeof(float) * nf);
  if (e == cudaSuccess) e = cudaMalloc(&p->nuts_lp, sizeof(double) * (p->max_chains > 0 ? p->max_chains : 1));
  if (e == cudaSuccess) e = cudaMalloc(&p->nuts_st, sizeof(NutsChain) * (p->max_chains > 0 ? p->max_chains : 1));
  if (e == cudaSuccess) e = cudaMalloc(&p->nuts_flags, sizeof(int) * 2);
  if (e == cudaSuccess) e = cudaMallocHost(&p->nuts_hflags, sizeof(int) * 2);
  return e;
}

static NutsArgs nuts_args(mt_problem *p) {
  const size_t CP = (size_t)(p->max_chains > 0 ? p->max_chains : 1) * p->P;
  float *w = p->nuts_ws;
  NutsArgs n{};
  float **f[] = {&n.thL, &n.pL, &n.gL, &n.thR, &n.pR, &n.gR, &n.thw, &n.pw, &n.gw, &n.ths, &n.gs,
                 &n.rho, &n.rhos, &n.tmp};
  for (size_t k = 0; k < sizeof(f) / sizeof(f[0]); k++) *f[k] = w + k * CP;
  n.rck = w + 16 * CP;
  n.rsck = n.rck + MT_NUTS_MAX_DEPTH * CP;
  n.lpw_out = p->nuts_lp;
  n.st = p->nuts_st;
  n.any_active = p->nuts_flags;
  n.any_sub = p->nuts_flags + 1;
  n.minv = p->d_minv;
  return n;
}

cudaError_t run_nuts(mt_problem *p, int C, float *x, double *logp, float *grad, const float *eps, int max_depth,
                     uint64_t seed, uint64_t iter, uint64_t chain_offset, float *accept_stat, int32_t *depth,
                     int32_t *n_leaves, int32_t *status, cudaStream_t s, std::string &why) {
  cudaError_t e = nuts_workspace(p);
  if (e != cudaSuccess) return e;
  // the checkpoint stride in k_nuts_leaf is C·P: pack the per-chain arrays at this C
  NutsArgs n = nuts_args(p);
  {
    const size_t CP = (size_t)C * p->P;
    float *w = p->nuts_ws;
    float **f[] = {&n.thL, &n.pL, &n.gL, &n.thR, &n.pR, &n.gR, &n.thw, &n.pw, &n.gw, &n.ths, &n.gs,
                   &n.rho, &n.rhos, &n.tmp};
    for (size_t k = 0; k < sizeof(f) / sizeof(f[0]); k++) *f[k] = w + k * CP;
    n.rck = w + 16 * CP;
    n.rsck = n.rck + MT_NUTS_MAX_DEPTH * CP;
  }
  FinishArgs a = base_args(p, C);
  a.eps = eps;
  k_nuts_begin<<<C, MT_THREADS, 0, s>>>(a, n, x, logp, grad, seed, iter, chain_offset);
  p->all_launches++;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  for (int j = 0; j < max_depth; j++) {
    if ((e = cudaMemsetAsync(p->nuts_flags, 0, sizeof(int) * 2, s)) != cudaSuccess) return e;
    k_nuts_subtree_begin<<<C, MT_THREADS, 0, s>>>(n, p->P, j, seed, iter, chain_offset);
    p->all_launches++;
    for (int t = 0; t < (1 << j); t++) {
      k_nuts_kick<<<C, MT_THREADS, 0, s>>>(a, n);
      p->all_launches++;
      if ((e = launch_trace(p, TRACE_LL, C, p->d_H, p->d_band, p->d_G, p->d_ll, nullptr, nullptr, s)) != cudaSuccess)
        return e;
      if ((e = launch_finish(p, FIN_PLAIN, C, n.thw, n.gw, n.lpw_out, nullptr, nullptr, nullptr, nullptr, s)) !=
          cudaSuccess)
        return e;
      if (p->comm && comm_allreduce_logp_grad(p, C, n.lpw_out, n.gw, s, why) != cudaSuccess) return cudaErrorUnknown;
      if ((e = cudaMemsetAsync(p->nuts_flags + 1, 0, sizeof(int), s)) != cudaSuccess) return e;
      k_nuts_leaf<<<C, MT_THREADS, 0, s>>>(a, n, t, seed, iter, chain_offset);
      p->all_launches++;
      if (j >= 3 && t + 1 < (1 << j)) {   // every chain's subtree stopped: skip the rest of it
        if ((e = cudaMemcpyAsync(p->nuts_hflags + 1, p->nuts_flags + 1, sizeof(int), cudaMemcpyDeviceToHost, s)) !=
            cudaSuccess)
          return e;
        if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
        if (!p->nuts_hflags[1]) break;
      }
    }
    k_nuts_merge<<<C, MT_THREADS, 0, s>>>(n, p->P, j, max_depth, x, logp, grad, seed, iter, chain_offset);
    p->all_launches++;
    if ((e = cudaMemcpyAsync(p->nuts_hflags, p->nuts_flags, sizeof(int), cudaMemcpyDeviceToHost, s)) != cudaSuccess)
      return e;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
    if (!p->nuts_hflags[0]) break;
  }
  k_nuts_end<<<(C + 255) / 256, 256, 0, s>>>(n, C, accept_stat, depth, n_leaves, status);
  p->all_launches++;
  return cudaGetLastError();
}
