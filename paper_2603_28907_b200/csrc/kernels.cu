// kernels.cu — K1 (latent -> heights), K3 (chain rule + CAR prior + logpost,
// fused leapfrog kick/drift + next heights), the few-chain multi-block K3 and
// kicks, sampled-r variants, HMC begin/end (Philox momenta, Metropolis), raw
// Philox, FP32 peak microbenchmark, and the launchers of all per-chain kernels
// (NUTS: nuts.cu; non-centred: ncp.cu; shared helpers: chain_common.cuh).
// B200 / sm_100a.
//
// All per-chain kernels use one 256-thread block per chain: a chain's state is
// P = 2 n_x n_y <= 8192 floats, so a block streams it once (coalesced), does
// the 5-point periodic stencil from shared memory and reduces per-chain
// scalars without atomics.
#include <curand_philox4x32_x.h>
#include <math.h>

#include "mt_internal.cuh"

#include "chain_common.cuh"

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
  macc *Gt = const_cast<macc *>(a.G);
  float *gc = a.grad + (size_t)c * a.P;
  float *pc = MODE != FIN_PLAIN ? a.mom + (size_t)c * a.P : nullptr;
  const float eps = MODE != FIN_PLAIN ? a.eps[c] : 0.f;
  BlockRed v = {3.0e38f, -3.0e38f, 3.0e38f, -3.0e38f, 0.0, 0.0, 0};
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    const int i = k / ny, j = k - i * ny;
    float x0 = xs[k], x1 = xs[N + k];
    NodeH h = node_heights(x0, x1, a.inv_sigma[0], a.inv_sigma[1], a.z_top, true);
    const size_t t0 = tix(c, 0, k, N), t1 = tix(c, 1, k, N);
    const double G0 = dq_g(Gt[t0]), G1 = dq_g(Gt[t1]);
    Gt[t0] = 0;
    Gt[t1] = 0;
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
    double lp = dq_ll(a.ll[c]) + (a.prior_on ? -0.5 * r.s0 + a.prior_const : 0.0);
    a.ll[c] = 0;
    a.logp[c] = lp;
    int bad = r.bad || !isfinite(lp);
    if (a.status) a.status[c] = bad ? MT_STATUS_NONFINITE : 0;
    if (MODE == FIN_STEP) a.band[c] = make_float4(r.mn0, r.mx0, r.mn1, r.mx1);
    if (MODE == FIN_LAST && a.kin) a.kin[c] = (float)r.s1;
  }
}

// ---------------------------------------------------------------------------
// K3, group-tiled (fixed r, centred, C >= 16): block = one 32-chain group x a
// tile of FG_T consecutive nodes, lane = chain.  The chain-interleaved streams
// (∂ℓ/∂H in, its zeroing, next H / Hlo out) are then 256-B / 128-B coalesced
// lines instead of one 8-B / 4-B word per 256-B / 128-B stride, and the
// caller-layout rows (x, p in; x, p, grad out) go through shared memory with a
// 33-float node stride (conflict-free both ways).  The x window carries ny
// halo nodes on each side, so the torus stencil's four neighbours of every
// tile node are in it (window position = node - k0 + ny, mod N).  Per-chain
// sums (prior quadratic, kinetic, band, non-finite flag) go to per-tile
// partials; the group's last block (ticket) reduces them in tile order, so
// the result does not depend on block scheduling (R30).  Per-node arithmetic
// is k_finish's, operation for operation.
// ---------------------------------------------------------------------------
// nodes per tile: 64 for the plain K3, 32 for the fused leapfrog (STEP / LAST hold
// momenta and gradient tiles too: 32-node tiles keep 4 blocks per SM, 0.35 vs 0.41 ms)
template <int MODE> struct FgTile { static constexpr int T = MODE == FIN_PLAIN ? 64 : 32; };
struct FinPart {   // 48 B: float4 band | double2 (prior, kinetic) sums | non-finite flag
  float mn0, mx0, mn1, mx1;
  double s0, s1;
  int bad, pad[3];
};

template <int MODE>
__global__ void __launch_bounds__(MT_THREADS, 4) k_finish_g(FinishArgs a, FinPart *part, unsigned *ticket) {
  constexpr int FG_T = FgTile<MODE>::T;
  extern __shared__ float fsm[];
  const int N = a.N, ny = a.ny, P = a.P;
  const int tile = blockIdx.x, g = blockIdx.y, ntile = gridDim.x;
  const int k0 = tile * FG_T, nt = min(FG_T, N - k0);
  const int W = FG_T + 2 * ny;                                   // x window (halo ny each side)
  float *xs = fsm;                                               // [2][W][33]
  float *ms = xs + 2 * W * 33;                                   // [2][FG_T][33] momenta
  float *gs = ms + (MODE != FIN_PLAIN ? 2 * FG_T * 33 : 0);      // [2][FG_T][33] gradient
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c0 = g * 32, nc = min(32, a.C - c0);
  const bool act = lane < nc;
  const int c = c0 + lane;
  // this thread's ∂ℓ/∂H words first (long-latency, independent of shared memory)
  macc *Gt = const_cast<macc *>(a.G);
  macc gq0[FG_T / 8], gq1[FG_T / 8];
#pragma unroll
  for (int m = 0; m < FG_T / 8; m++) {
    const int q = warp + 8 * m;
    const size_t t0 = ((size_t)(2 * g) * N + k0 + q) * 32 + lane;
    gq0[m] = (q < nt && act) ? Gt[t0] : 0;
    gq1[m] = (q < nt && act) ? Gt[t0 + (size_t)N * 32] : 0;
  }
  // x window and momenta rows, 8 loads in flight per thread
  for (int cc = warp; cc < nc; cc += MT_THREADS / 32) {
    const float *xc = a.xin + (size_t)(c0 + cc) * P;
    for (int q0 = 0; q0 < W; q0 += 128) {
      float v[2][4];
#pragma unroll
      for (int l = 0; l < 2; l++)
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const int q = q0 + lane + 32 * u;
          int k = (k0 - ny + q) % N;
          k += k < 0 ? N : 0;
          v[l][u] = q < W ? xc[l * N + k] : 0.f;
        }
#pragma unroll
      for (int l = 0; l < 2; l++)
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const int q = q0 + lane + 32 * u;
          if (q < W) xs[(l * W + q) * 33 + cc] = v[l][u];
        }
    }
    if (MODE != FIN_PLAIN) {
      const float *pc = a.mom + (size_t)(c0 + cc) * P;
      float v[2][FG_T / 32];
#pragma unroll
      for (int l = 0; l < 2; l++)
#pragma unroll
        for (int u = 0; u < FG_T / 32; u++) {
          const int q = lane + 32 * u;
          v[l][u] = q < nt ? pc[l * N + k0 + q] : 0.f;
        }
#pragma unroll
      for (int l = 0; l < 2; l++)
#pragma unroll
        for (int u = 0; u < FG_T / 32; u++) {
          const int q = lane + 32 * u;
          if (q < nt) ms[(l * FG_T + q) * 33 + cc] = v[l][u];
        }
    }
  }
  __syncthreads();
  const float eps = (MODE != FIN_PLAIN && act) ? a.eps[c] : 0.f;
  float mn0 = 3.0e38f, mx0 = -3.0e38f, mn1 = 3.0e38f, mx1 = -3.0e38f;
  double s0 = 0.0, s1 = 0.0;
  int bad = 0;
  float xn0[FG_T / 8], xn1[FG_T / 8];
#pragma unroll
  for (int m = 0; m < FG_T / 8; m++) {
    const int q = warp + 8 * m;
    xn0[m] = xn1[m] = 0.f;
    if (q >= nt || !act) continue;
    const int k = k0 + q, j = k % ny, pos = q + ny;
    const float x0 = xs[pos * 33 + lane], x1 = xs[(W + pos) * 33 + lane];
    const JacF h = node_jac32(x0, x1, a.inv_sigma[0], a.inv_sigma[1], a.z_top);
    const size_t t0 = ((size_t)(2 * g) * N + k) * 32 + lane, t1 = t0 + (size_t)N * 32;
    const double G0 = dq_g(gq0[m]), G1 = dq_g(gq1[m]);
    Gt[t0] = 0;
    Gt[t1] = 0;
    double gx0 = (double)G0 * h.J0 + (double)G1 * h.J10;
    double gx1 = (double)G1 * h.J11;
    if (a.prior_on) {
      const int pip = pos + ny, pim = pos - ny;   // (i ± 1, j), torus-wrapped by the window
      const int pjp = j + 1 == ny ? pos - (ny - 1) : pos + 1, pjm = j == 0 ? pos + (ny - 1) : pos - 1;
#pragma unroll
      for (int l = 0; l < 2; l++) {
        const float *xl = xs + l * W * 33 + lane;
        double xv = xl[pos * 33];
        double Qx = 4.0 * xv - (double)a.car_r[l] * ((double)xl[pip * 33] + xl[pim * 33] + xl[pjp * 33] + xl[pjm * 33]);
        s0 += xv * Qx;
        if (l == 0) gx0 -= Qx; else gx1 -= Qx;
      }
    }
    const float g0f = (float)gx0, g1f = (float)gx1;
    bad |= !(isfinite(g0f) && isfinite(g1f));
    gs[q * 33 + lane] = g0f;
    gs[(FG_T + q) * 33 + lane] = g1f;
    if (MODE == FIN_STEP) {  // close this step's half kick, open the next: p += ε g; x += ε p
      const float p0 = ms[q * 33 + lane] + eps * g0f, p1 = ms[(FG_T + q) * 33 + lane] + eps * g1f;
      ms[q * 33 + lane] = p0;
      ms[(FG_T + q) * 33 + lane] = p1;
      const float a0 = x0 + eps * mi(a, k) * p0, a1 = x1 + eps * mi(a, N + k) * p1;
      xn0[m] = a0;
      xn1[m] = a1;
      NodeH hn = node_heights(a0, a1, a.inv_sigma[0], a.inv_sigma[1], a.z_top, false);
      a.H[t0] = hn.H0;
      a.H[t1] = hn.H1;
      a.Hlo[t0] = hn.L0;
      a.Hlo[t1] = hn.L1;
      mn0 = fminf(mn0, hn.H0); mx0 = fmaxf(mx0, hn.H0);
      mn1 = fminf(mn1, hn.H1); mx1 = fmaxf(mx1, hn.H1);
    } else if (MODE == FIN_LAST) {  // final half kick
      const float p0 = ms[q * 33 + lane] + 0.5f * eps * g0f, p1 = ms[(FG_T + q) * 33 + lane] + 0.5f * eps * g1f;
      ms[q * 33 + lane] = p0;
      ms[(FG_T + q) * 33 + lane] = p1;
      s1 += 0.5 * ((double)mi(a, k) * p0 * p0 + (double)mi(a, N + k) * p1 * p1);
    }
  }
  // per-chain partials of this tile: the 8 warps' values, summed in warp order
  __shared__ float4 wb[MT_THREADS / 32][32];
  __shared__ double2 ws[MT_THREADS / 32][32];
  __shared__ int wbad[MT_THREADS / 32][32];
  __shared__ int last;
  wb[warp][lane] = make_float4(mn0, mx0, mn1, mx1);
  ws[warp][lane] = make_double2(s0, s1);
  wbad[warp][lane] = bad;
  __syncthreads();   // (all window reads done: the new x may overwrite it)
  if (MODE == FIN_STEP) {
#pragma unroll
    for (int m = 0; m < FG_T / 8; m++) {
      const int q = warp + 8 * m;
      if (q < nt && act) {
        xs[(q + ny) * 33 + lane] = xn0[m];
        xs[(W + q + ny) * 33 + lane] = xn1[m];
      }
    }
  }
  if (warp == 0) {
    float4 b = wb[0][lane];
    double2 sm = ws[0][lane];
    int bb = wbad[0][lane];
    for (int w = 1; w < MT_THREADS / 32; w++) {
      const float4 o = wb[w][lane];
      b = make_float4(fminf(b.x, o.x), fmaxf(b.y, o.y), fminf(b.z, o.z), fmaxf(b.w, o.w));
      sm.x += ws[w][lane].x;
      sm.y += ws[w][lane].y;
      bb |= wbad[w][lane];
    }
    FinPart *pp = part + ((size_t)g * ntile + tile) * 32 + lane;
    *reinterpret_cast<float4 *>(pp) = b;
    *(reinterpret_cast<double2 *>(pp) + 1) = sm;
    *(reinterpret_cast<int *>(pp) + 8) = bb;
    __threadfence();
  }
  __syncthreads();
  // write back the caller-layout rows (coalesced along nodes)
  for (int cc = warp; cc < nc; cc += MT_THREADS / 32) {
    const size_t row = (size_t)(c0 + cc) * P;
#pragma unroll
    for (int l = 0; l < 2; l++)
      for (int q = lane; q < nt; q += 32) {
        const int o = l * N + k0 + q;
        a.grad[row + o] = gs[(l * FG_T + q) * 33 + cc];
        if (MODE != FIN_PLAIN) a.mom[row + o] = ms[(l * FG_T + q) * 33 + cc];
        if (MODE == FIN_STEP || (MODE == FIN_LAST && a.xin != a.x)) a.x[row + o] = xs[(l * W + q + ny) * 33 + cc];
      }
  }
  if (threadIdx.x == 0) last = atomicAdd(ticket + g, 1u) == (unsigned)(ntile - 1);
  __syncthreads();
  if (!last || warp != 0) return;
  __threadfence();
  FinPart r = {3.0e38f, -3.0e38f, 3.0e38f, -3.0e38f, 0.0, 0.0, 0, 0};
  for (int t = 0; t < ntile; t++) {   // tile order: independent of which block finished last
    const FinPart *pp = part + ((size_t)g * ntile + t) * 32 + lane;
    const float4 b = __ldcg(reinterpret_cast<const float4 *>(pp));
    const double2 s = __ldcg(reinterpret_cast<const double2 *>(pp) + 1);
    const int bb = __ldcg(reinterpret_cast<const int *>(pp) + 8);
    r.mn0 = fminf(r.mn0, b.x); r.mx0 = fmaxf(r.mx0, b.y);
    r.mn1 = fminf(r.mn1, b.z); r.mx1 = fmaxf(r.mx1, b.w);
    r.s0 += s.x; r.s1 += s.y; r.bad |= bb;
  }
  if (lane == 0) ticket[g] = 0;
  if (!act) return;
  const double lp = dq_ll(a.ll[c]) + (a.prior_on ? -0.5 * r.s0 + a.prior_const : 0.0);
  a.ll[c] = 0;
  a.logp[c] = lp;
  if (a.status) a.status[c] = (r.bad || !isfinite(lp)) ? MT_STATUS_NONFINITE : 0;
  if (MODE == FIN_STEP) a.band[c] = make_float4(r.mn0, r.mx0, r.mn1, r.mx1);
  if (MODE == FIN_LAST && a.kin) a.kin[c] = (float)r.s1;
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
  macc *Gt = const_cast<macc *>(a.G);
  BlockRed v = {3.0e38f, -3.0e38f, 3.0e38f, -3.0e38f, 0.0, 0.0, 0};
  for (int k = blockIdx.y * blockDim.x + threadIdx.x; k < N; k += gridDim.y * blockDim.x) {
    const int i = k / ny, j = k - i * ny;
    const float x0 = xc[k], x1 = xc[N + k];
    const NodeH h = node_heights(x0, x1, a.inv_sigma[0], a.inv_sigma[1], a.z_top, true);
    const size_t t0 = tix(c, 0, k, N), t1 = tix(c, 1, k, N);
    const double G0 = dq_g(Gt[t0]), G1 = dq_g(Gt[t1]);
    Gt[t0] = 0;
    Gt[t1] = 0;
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
    const double lp = dq_ll(a.ll[c]) + (a.prior_on ? -0.5 * rd[0] + a.prior_const : 0.0);
    a.ll[c] = 0;
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
                                                          uint64_t iter, uint64_t chain_offset,
                                                          const uint64_t *iter_dev) {
  const int c = blockIdx.x, N = a.N, P = a.P;
  if (iter_dev) iter = *iter_dev;   // device step counter (graph replay)
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
                                                        int32_t *accepted, const uint64_t *iter_dev) {
  __shared__ int s_acc;
  if (iter_dev) iter = *iter_dev;
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
  // clock span over every block resident on SM 0 (clock64 is per SM): block 0
  // alone finishes early under oldest-first warp scheduling
  unsigned sm;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  if (sm == 0 && threadIdx.x == 0) {
    atomicMin((unsigned long long *)&cycles[0], (unsigned long long)t0);
    atomicMax((unsigned long long *)&cycles[1], (unsigned long long)t1);
  }
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
  macc *Gt = const_cast<macc *>(a.G);
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
    const double G0 = dq_g(Gt[t0]), G1 = dq_g(Gt[t1]);
    Gt[t0] = 0;
    Gt[t1] = 0;
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
    double lp = dq_ll(a.ll[c]);
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
    a.ll[c] = 0;
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

FinishArgs base_args(mt_problem *p, int C) {
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

bool use_fg(const mt_problem *p, int C) {
  return p->d_fin_part != nullptr && C >= 16 && !p->sample_r && !p->ncp && !use_mb(p, C);
}

template <int MODE>
static cudaError_t launch_fg(mt_problem *p, const FinishArgs &a, int C, cudaStream_t s) {
  static size_t done[64] = {};
  constexpr int FG_T = FgTile<MODE>::T;
  const int W = FG_T + 2 * p->ny;
  const size_t smem = sizeof(float) * 33 * (2 * (size_t)W + 2 * FG_T * (MODE == FIN_PLAIN ? 1 : 2));
  const int dv = p->device & 63;
  if (smem > 32 * 1024 && done[dv] < smem) {   // (dynamic + 9 KB static must fit the attribute)
    cudaError_t e = cudaFuncSetAttribute(k_finish_g<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    done[dv] = smem;
  }
  const dim3 grid((unsigned)((p->N + FG_T - 1) / FG_T), (unsigned)((C + 31) / 32));
  k_finish_g<MODE><<<grid, MT_THREADS, smem, s>>>(a, reinterpret_cast<FinPart *>(p->d_fin_part), p->d_fin_ticket);
  p->all_launches++;
  return cudaGetLastError();
}

cudaError_t launch_finish(mt_problem *p, int mode, int C, float *x, float *grad, double *logp,
                          int32_t *status, float *mom, const float *eps, float *kin,
                          cudaStream_t s, const float *xin) {
  if (C <= 0) return cudaSuccess;
  if (mode != FIN_PLAIN && mode != FIN_STEP && mode != FIN_LAST) return cudaErrorInvalidValue;
  FinishArgs a = base_args(p, C);
  a.x = x; a.grad = grad; a.logp = logp; a.status = status; a.mom = mom; a.eps = eps; a.kin = kin;
  a.xin = xin ? xin : x;
  if (use_fg(p, C)) {
    if (mode == FIN_PLAIN) return launch_fg<FIN_PLAIN>(p, a, C, s);
    if (mode == FIN_STEP) return launch_fg<FIN_STEP>(p, a, C, s);
    return launch_fg<FIN_LAST>(p, a, C, s);
  }
  if (a.xin != x) return cudaErrorInvalidValue;   // (only the group-tiled K3 reads a separate x)
  if (use_mb(p, C)) {   // few chains: several blocks per chain (unfused leapfrog)
    if (mode != FIN_PLAIN) return cudaErrorInvalidValue;
    k_finish_mb<<<dim3(C, mb_blocks(p, C)), MT_THREADS, 0, s>>>(a, mb_scratch(p));
    p->all_launches++;
    return cudaGetLastError();
  }
  if (p->ncp) {   // unfused: the API drives kicks / drifts separately (k_ncp_kick)
    if (mode != FIN_PLAIN) return cudaErrorInvalidValue;
    launch_ncp_finish(p, a, C, s);
    p->all_launches++;
    return cudaGetLastError();
  }
  size_t smem = (size_t)p->P * sizeof(float);
  if (mode < 0 || mode > 2) return cudaErrorInvalidValue;
  // shared-memory opt-in, once per (device, mode); a failure is returned (and not recorded)
  static bool attr[64][3] = {}, attr_r[64][3] = {};
  const int dv = p->device & 63;
  if (smem > 48 * 1024 && !(p->sample_r ? attr_r : attr)[dv][mode]) {
    cudaError_t e;
    if (p->sample_r)
      e = cudaFuncSetAttribute(mode == FIN_PLAIN ? (const void *)k_finish_r<FIN_PLAIN>
                               : mode == FIN_STEP ? (const void *)k_finish_r<FIN_STEP> : (const void *)k_finish_r<FIN_LAST>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    else
      e = cudaFuncSetAttribute(mode == FIN_PLAIN ? (const void *)k_finish<FIN_PLAIN>
                               : mode == FIN_STEP ? (const void *)k_finish<FIN_STEP> : (const void *)k_finish<FIN_LAST>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    if (e != cudaSuccess) return e;
    (p->sample_r ? attr_r : attr)[dv][mode] = true;
  }
  if (p->sample_r) {
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
  if (p->ncp) {   // non-centred: kick / drift in z, heights of x = U z
    launch_ncp_kick(p, mode, a, C, s);
    p->all_launches += mode != KICK_HALF_LAST ? 2 : 1;
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
                                       chain_offset, p->d_iter);
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
                                     iter, chain_offset, acc_prob, accepted, p->d_iter);
  p->all_launches++;
  if (p->d_iter) {   // the step's Philox iteration is used: advance the device counter
    cudaError_t e = launch_counter_add(p->d_iter, nullptr, s);
    if (e != cudaSuccess) return e;
    p->all_launches++;
  }
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

// Fixed-point accumulators -> the caller's ∂ℓ/∂H [C][2N] fp32 and ℓ [C] fp64 (debug /
// parity entry mt_loglik_heights); the accumulators are cleared.
__global__ void k_take_acc(int C, int N, macc *G, macc *ll, float *dldH, double *llo) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < C) {
    llo[t] = dq_ll(ll[t]);
    ll[t] = 0;
  }
  if (t >= (int64_t)C * 2 * N) return;
  const int c = (int)(t / (2 * N)), m = (int)(t - (int64_t)c * 2 * N);
  const size_t ti = tix(c, m / N, m % N, N);
  dldH[t] = (float)dq_g(G[ti]);
  G[ti] = 0;
}

cudaError_t launch_take_acc(mt_problem *p, int C, float *dldH, double *ll, cudaStream_t s) {
  if (C <= 0) return cudaSuccess;
  const int64_t n = (int64_t)C * 2 * p->N;
  k_take_acc<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(C, p->N, p->d_G, p->d_ll, dldH, ll);
  p->all_launches++;
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
  cudaMalloc(&cyc, 2 * sizeof(long long));
  const long long cyc_init[2] = {0x7fffffffffffffffLL, 0};
  int blocks = prop.multiProcessorCount * 4, threads = 512, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_ffma<<<blocks, threads>>>(out, 64, 1.0000001f, 1e-7f, cyc);  // warm-up
  double best = 0, best_mhz = 0;
  for (int rep = 0; rep < 10; rep++) {
    cudaMemcpy(cyc, cyc_init, sizeof(cyc_init), cudaMemcpyHostToDevice);
    cudaEventRecord(e0);
    k_ffma<<<blocks, threads>>>(out, iters, 1.0000001f, 1e-7f, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    long long span[2] = {0, 0};
    cudaMemcpy(span, cyc, sizeof(span), cudaMemcpyDeviceToHost);
    long long cycles = span[1] - span[0];
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
