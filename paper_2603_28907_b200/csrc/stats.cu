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

__global__ void k_welford(int64_t n, const float4 *x, float4 *mean, float4 *m2, float inv_cnt) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  float4 v = x[t], m = mean[t], s = m2[t];
  float d0 = v.x - m.x, d1 = v.y - m.y, d2 = v.z - m.z, d3 = v.w - m.w;
  m.x += d0 * inv_cnt; m.y += d1 * inv_cnt; m.z += d2 * inv_cnt; m.w += d3 * inv_cnt;
  s.x += d0 * (v.x - m.x); s.y += d1 * (v.y - m.y); s.z += d2 * (v.z - m.z); s.w += d3 * (v.w - m.w);
  mean[t] = m;
  m2[t] = s;
}

__global__ void k_welford_scalar(int64_t n, const float *x, float *mean, float *m2, float inv_cnt) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
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
          reinterpret_cast<float4 *>(m2), inv);
    } else {
      k_welford_scalar<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, x, mean, m2, inv);
    }
    p->all_launches++;
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
