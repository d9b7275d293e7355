// nuts.cu — batched lockstep NUTS (reading R26):
// tree state and checkpoints per chain, one leaf (= one evaluation of every
// chain) per step, finished chains idle.  B200 / sm_100a.
#include "chain_common.cuh"

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
      const int leaf = (1 << j) - 1 + t;
      if (p->nuts_rec_th && leaf < p->nuts_rec_max) {   // debug / parity record of the leaf (mt_nuts_record)
        const size_t CP = (size_t)C * p->P;
        if ((e = cudaMemcpyAsync(p->nuts_rec_th + leaf * CP, n.thw, sizeof(float) * CP, cudaMemcpyDeviceToDevice, s)) !=
                cudaSuccess ||
            (e = cudaMemcpyAsync(p->nuts_rec_g + leaf * CP, n.gw, sizeof(float) * CP, cudaMemcpyDeviceToDevice, s)) !=
                cudaSuccess ||
            (e = cudaMemcpyAsync(p->nuts_rec_lp + (size_t)leaf * C, n.lpw_out, sizeof(double) * C,
                                 cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
          return e;
      }
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

