// stats.cu — K5: per-iteration sampler statistics.
//  * acceptance: Σ_c round(accept_prob_c · 2^32) and C as int64, so the
//    cross-rank sum is exact and order-independent (HP9) and the dual-averaging
//    step size is bit-identical for any GPU count;
//  * Welford running mean / M2 of x per (chain, parameter) over sampling
//    iterations;
//  * R-hat partial sums over this rank's chains: Σ_c m̄_c, Σ_c m̄_c², Σ_c s²_c
//    (classic between/within decomposition, reading R21).
#include "mt_internal.cuh"

__global__ void k_accept_sum(int C, const float *acc, unsigned long long *out) {
  __shared__ unsigned long long sh[MT_THREADS];
  unsigned long long v = 0;
  for (int c = threadIdx.x; c < C; c += blockDim.x)
    v += (unsigned long long)llrint((double)acc[c] * 4294967296.0);
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    atomicAdd(out, sh[0]);
    atomicAdd(out + 1, (unsigned long long)C);
  }
}

__global__ void k_welford(int64_t n, const float4 *x, float4 *mean, float4 *m2, float inv_cnt,
                          const int32_t *nprev_dev) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  if (nprev_dev) inv_cnt = 1.0f / (float)(*nprev_dev + 1);   // device step counter (graph replay)
  float4 v = x[t], m = mean[t], s = m2[t];
  float d0 = v.x - m.x, d1 = v.y - m.y, d2 = v.z - m.z, d3 = v.w - m.w;
  m.x += d0 * inv_cnt; m.y += d1 * inv_cnt; m.z += d2 * inv_cnt; m.w += d3 * inv_cnt;
  s.x += d0 * (v.x - m.x); s.y += d1 * (v.y - m.y); s.z += d2 * (v.z - m.z); s.w += d3 * (v.w - m.w);
  mean[t] = m;
  m2[t] = s;
}

__global__ void k_welford_scalar(int64_t n, const float *x, float *mean, float *m2, float inv_cnt,
                                 const int32_t *nprev_dev) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  if (nprev_dev) inv_cnt = 1.0f / (float)(*nprev_dev + 1);
  float v = x[t], m = mean[t];
  float d = v - m;
  m += d * inv_cnt;
  mean[t] = m;
  m2[t] += d * (v - m);
}

// one thread per parameter, loop over chains (coalesced across threads)
__global__ void k_rhat_partials(int C, int P, const float *mean, const float *m2, double inv_nm1,
                                double *out) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= P) return;
  double s1 = 0, s2 = 0, sv = 0;
  for (int c = 0; c < C; c++) {
    double m = mean[(size_t)c * P + k];
    s1 += m;
    s2 += m * m;
    sv += (double)m2[(size_t)c * P + k] * inv_nm1;
  }
  out[k] = s1;
  out[P + k] = s2;
  out[2 * P + k] = sv;
}

// nested R̂ partial sums (Margossian et al.'s super-chains; reading
// R21b): chains [kM, (k+1)M) form super-chain k (same start).  Per
// parameter and super-chain: m_k = mean of its chain means; W_k = W̃_k + B̃_k,
// the mean within-chain variance (m2/(n-1); 0 for one draw per chain, the
// paper's keep-last protocol) plus the variance of its chain means (M-1 in the
// denominator).  out [3][P] = (Σ_k m_k, Σ_k m_k², Σ_k W_k) over this rank's
// super-chains; a SUM over ranks and the host give B = var_k m_k, W = mean_k W_k,
// nested R̂ = sqrt(1 + B/W).
__global__ void k_nested_rhat_partials(int C, int P, int M, const float *mean, const float *m2,
                                       double inv_nm1, double *out) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= P) return;
  double s1 = 0, s2 = 0, sw = 0;
  for (int c0 = 0; c0 + M <= C; c0 += M) {
    double mk = 0, wt = 0;
    for (int c = c0; c < c0 + M; c++) {
      mk += mean[(size_t)c * P + k];
      wt += (double)m2[(size_t)c * P + k] * inv_nm1;
    }
    mk /= M;
    wt /= M;
    double bt = 0;
    if (M > 1) {
      for (int c = c0; c < c0 + M; c++) {
        const double d = mean[(size_t)c * P + k] - mk;
        bt += d * d;
      }
      bt /= (M - 1);
    }
    s1 += mk;
    s2 += mk * mk;
    sw += wt + bt;
  }
  out[k] = s1;
  out[P + k] = s2;
  out[2 * P + k] = sw;
}

cudaError_t launch_nested_rhat_partials(mt_problem *p, int C, int M, const float *mean, const float *m2,
                                        int32_t n, double *out, cudaStream_t s) {
  double inv = n > 1 ? 1.0 / (n - 1) : 0.0;
  k_nested_rhat_partials<<<(p->P + 255) / 256, 256, 0, s>>>(C, p->P, M, mean, m2, inv, out);
  p->all_launches++;
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// posterior summaries (reading R27): from the
// current draws x [C][P] and their heights H (chain-interleaved, from K1):
//   acc[0]                      number of draws accumulated
//   acc[1 .. 2N]                Σ H_l(node)              -> posterior-mean heights
//   acc[1+2N .. 1+3N)           #draws with H1 - H0 > gap (air-gap thickness exceedance)
//   then Σ D, Σ D² per layer l in {muck, air, rock}, node, voxel k (layer-indicator
//   tomography): D^(l) = ς(H_l - z_k) - ς(H_{l-1} - z_k) with
//   ς(u) = 1/(1+e^{-u/γ}), γ = 1 m, H_{-1} = 0 (floor), H_2 = z_top, voxel
//   columns at the nodes, z_k = k Δz, Δz = z_top/n_z.
// Block = one node; thread = one voxel of its column; loop over chains.
__global__ void k_summary_update(int C, int N, int nz, float z_top, float gap, const float *H,
                                 double *acc) {
  const int n = blockIdx.x;
  const double dz = (double)z_top / nz;
  double sH0 = 0, sH1 = 0, sgap = 0;
  for (int k = threadIdx.x; k < nz; k += blockDim.x) {
    const double z = k * dz;
    double sd[3] = {0, 0, 0}, sd2[3] = {0, 0, 0};
    for (int c = 0; c < C; c++) {
      const double h0 = H[tix(c, 0, n, N)], h1 = H[tix(c, 1, n, N)];
      const double sf = 1.0 / (1.0 + exp(z)), s0 = 1.0 / (1.0 + exp(-(h0 - z)));
      const double s1 = 1.0 / (1.0 + exp(-(h1 - z))), st = 1.0 / (1.0 + exp(-((double)z_top - z)));
      const double D[3] = {s0 - sf, s1 - s0, st - s1};
#pragma unroll
      for (int l = 0; l < 3; l++) {
        sd[l] += D[l];
        sd2[l] += D[l] * D[l];
      }
      if (k == 0) {
        sH0 += h0;
        sH1 += h1;
        sgap += (h1 - h0) > gap ? 1.0 : 0.0;
      }
    }
    double *accD = acc + 1 + 3 * (size_t)N;
#pragma unroll
    for (int l = 0; l < 3; l++) {
      accD[((size_t)l * N + n) * nz + k] += sd[l];
      accD[(3 * (size_t)N + (size_t)l * N + n) * nz + k] += sd2[l];
    }
  }
  if (threadIdx.x == 0) {
    acc[1 + n] += sH0;
    acc[1 + N + n] += sH1;
    acc[1 + 2 * N + n] += sgap;
    if (n == 0) acc[0] += C;
  }
}

// MAP draw: the highest log-posterior among the C current draws
// replaces map_x / map_logp when higher (ties keep the first).
__global__ void k_map_update(int C, int P, const float *x, const double *logp, float *map_x, double *map_logp) {
  __shared__ double bv[MT_THREADS];
  __shared__ int bi[MT_THREADS];
  double v = -INFINITY;
  int idx = -1;
  for (int c = threadIdx.x; c < C; c += blockDim.x)
    if (logp[c] > v) { v = logp[c]; idx = c; }
  bv[threadIdx.x] = v;
  bi[threadIdx.x] = idx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int t = 1; t < (int)blockDim.x; t++)
      if (bv[t] > v || (bv[t] == v && bi[t] >= 0 && (idx < 0 || bi[t] < idx))) { v = bv[t]; idx = bi[t]; }
    bi[0] = (idx >= 0 && v > *map_logp) ? idx : -1;
    if (bi[0] >= 0) *map_logp = v;
  }
  __syncthreads();
  const int best = bi[0];
  if (best >= 0)
    for (int k = threadIdx.x; k < P; k += blockDim.x) map_x[k] = x[(size_t)best * P + k];
}

// f4 assembly (R27) from the accumulators of k_summary_update:
// out = [mean heights 2N | air-gap exceedance probability N | indicator std
// 3 N nz], std = sqrt(max(E[D²] - E[D]², 0)) per (unit, node, layer).
__global__ void k_summary_finalize(const double *acc, int N, int nz, double *out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n3 = 3 * (int64_t)N, nd = 3 * (int64_t)N * nz;
  if (t >= n3 + nd) return;
  const double n = acc[0];
  if (t < n3) {
    out[t] = acc[1 + t] / n;
  } else {
    const int64_t q = t - n3;
    const double m = acc[1 + n3 + q] / n, m2 = acc[1 + n3 + nd + q] / n;
    out[t] = sqrt(fmax(m2 - m * m, 0.0));
  }
}

cudaError_t launch_summary_finalize(mt_problem *p, int nz, const double *acc, double *out, cudaStream_t s) {
  const int64_t n = 3 * (int64_t)p->N * (1 + nz);
  k_summary_finalize<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(acc, p->N, nz, out);
  p->all_launches++;
  return cudaGetLastError();
}

cudaError_t launch_summary(mt_problem *p, int C, const float *x, const double *logp, int nz, float gap,
                           double *acc, float *map_x, double *map_logp, cudaStream_t s) {
  cudaError_t e = launch_heights(p, C, x, p->d_H, p->d_band, s);
  if (e != cudaSuccess) return e;
  k_summary_update<<<p->N, 64, 0, s>>>(C, p->N, nz, p->z_top, gap, p->d_H, acc);
  p->all_launches++;
  if (map_x && map_logp && logp) {
    k_map_update<<<1, MT_THREADS, 0, s>>>(C, p->P, x, logp, map_x, map_logp);
    p->all_launches++;
  }
  return cudaGetLastError();
}

// Device step counters (mt_set_step_counters): +1 on the Philox iteration and / or the
// Welford count, inside the captured step.
__global__ void k_counter_add(uint64_t *iter, int32_t *nprev) {
  if (iter) *iter += 1;
  if (nprev) *nprev += 1;
}

cudaError_t launch_counter_add(uint64_t *iter, int32_t *nprev, cudaStream_t s) {
  k_counter_add<<<1, 1, 0, s>>>(iter, nprev);
  return cudaGetLastError();
}

cudaError_t launch_stats(mt_problem *p, int C, const float *x, const float *acc, int32_t n_prev,
                         float *mean, float *m2, unsigned long long *acc_fixed, cudaStream_t s) {
  if (C <= 0) return cudaSuccess;
  if (acc && acc_fixed) {
    k_accept_sum<<<1, MT_THREADS, 0, s>>>(C, acc, acc_fixed);
    p->all_launches++;
  }
  if (mean && m2 && x) {
    int64_t n = (int64_t)C * p->P;
    float inv = 1.0f / (float)(n_prev + 1);
    if ((p->P & 3) == 0) {
      int64_t n4 = n / 4;
      k_welford<<<(unsigned)((n4 + 255) / 256), 256, 0, s>>>(
          n4, reinterpret_cast<const float4 *>(x), reinterpret_cast<float4 *>(mean),
          reinterpret_cast<float4 *>(m2), inv, p->d_nprev);
    } else {
      k_welford_scalar<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, x, mean, m2, inv, p->d_nprev);
    }
    p->all_launches++;
    if (p->d_nprev) {   // advance the device count after this update
      k_counter_add<<<1, 1, 0, s>>>(nullptr, p->d_nprev);
      p->all_launches++;
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_rhat_partials(mt_problem *p, int C, const float *mean, const float *m2,
                                 int32_t n, double *out, cudaStream_t s) {
  double inv = n > 1 ? 1.0 / (n - 1) : 0.0;
  k_rhat_partials<<<(p->P + 255) / 256, 256, 0, s>>>(C, p->P, mean, m2, inv, out);
  p->all_launches++;
  return cudaGetLastError();
}
