// voxel.cu — the paper's own forward model:
// voxel density grid, sigmoid layer indicators with partition-of-unity weights
// R̂(H), linearised expected counts λ̂ = λ(R0) + G(R̂ − R0) with the
// sparse sensitivity matrix G = ∂λ/∂R at R0, the Poisson
// likelihood of the exact model and its gradient back to the node heights.
// Readings R28/R29 of DESIGN.md fix what the paper leaves open.
//
// Setup (mt_voxel_model, once per reference geometry) runs on the host in
// double: an Amanatides-Woo walk of each ray through the voxel grid gives
// L_pv, then λ_p(R0) and G in CSR (rows = rays, for λ̂) and CSC (columns =
// voxels, for Gᵀ ∂ℓ/∂λ̂).  Per evaluation, three kernels replace the exact
// tracer between the heights (K1) and the chain rule / prior (K3):
//   V1 k_vx_rhat   ΔR_v = R̂_v(H) − R0_v                 (elementwise, sigmoids)
//   V2 k_vx_fwd    λ̂_p = λ0_p + Σ_v G_pv ΔR_v, ℓ_p, r_p = ∂ℓ/∂λ̂_p   (SpMV + epilogue)
//   V3 k_vx_bwd    ∂ℓ/∂H_l(node) = Σ_k (Σ_p G_pv r_p) ∂R̂_v/∂H_l     (SpMVᵀ + chain rule)
// V3 accumulates ∂ℓ/∂H (one warp per run of <= 512 CSC entries inside a node
// column, so the voxels next to a detector, crossed by every ray of it, are
// split over many warps; float atomics) into the same chain-interleaved
// workspace the exact tracer fills, so K3, the leapfrog/HMC/NUTS drivers,
// sampled r and ray sharding are unchanged.  Two layouts: chain lanes
// (C >= 16: a warp = one row / column × W = 32·VEC chains, VEC = 1, 2, 4
// chains per lane, every G entry loaded once per W chains, ΔR and r gathers
// are 128·VEC-byte lines) and row lanes (C < 16: 8-lane teams per CSR row,
// warp lanes over a CSC run, one chain at a time).  Only the layers within
// 24 γ of the chain group's height band are read (per-row layer-bucket
// offsets).  Grids are group-major (blockIdx.y = chain group).
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <thread>
#include <vector>

#include "mt_internal.cuh"

namespace {

constexpr int VX_WARPS = MT_THREADS / 32;
#ifndef VX_MINB
#define VX_MINB 5   // 48 registers, 5 blocks/SM: 3.82 vs 4.06 ms per Medium evaluation at 64
#endif
constexpr int VX_RPW_CL = 4;    // rays per warp, chain lanes
constexpr int VX_RPW_RL = 16;   // rays per warp, row lanes
constexpr float VX_ZC = 24.f;   // band margin in units of γ (skipped terms < 1e-9 λ0)
constexpr int VX_CH = 512;      // CSC entries per Gᵀ work item (balances the heavy voxels by the detectors)

struct VoxArgs {
  int C, N, ny, nz;
  int64_t R, ng;
  float dz, inv_gamma, z_top, tau;
  float rho_m, rho_a, rho_r;
  const float *H;          // chain-interleaved heights (tix layout)
  const float *R0;         // [ng]
  float *dR;               // CL: [grp][ng][32][VEC]; RL: [c][ng]
  float *r;                // CL: [grp][R][32][VEC];  RL: [c][R]
  const int64_t *rowptr;   // [R+1]
  const uint4 *kofs;       // [R]: 8 uint16 offsets (from the row start) of the first entry of layer >= b·kb
  int kb;                  // layers per offset bucket
  const int2 *csr;         // {voxel, G bits}
  const int64_t *colptr;   // [ng+1]
  const int2 *csc;         // {ray, G bits}
  const float2 *lc;        // {λ_p(R0), C_p}
  const VxItem *items;     // Gᵀ work items
  int64_t n_items;
  const float4 *band;      // per chain {min H0, max H0, min H1, max H1}
  float href_lo, href_hi;  // min H_ref,0 and max H_ref,1
  float zc;                // band margin (VX_ZC γ)
  int rpw;                 // rays per warp in V2
  int g0;                  // first chain group of this launch (blockIdx.y + g0)
  unsigned long long *gathered;   // optional: += ΔR bytes gathered by V2 (valid chains × 4 B per kept entry)
  macc *G;                 // ∂ℓ/∂H out (tix layout)
  macc *ll;                // [C] += Σ_p ℓ_p
};

__device__ __forceinline__ float warp_allsum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float sig(float u, float ig) { return 1.f / (1.f + __expf(-u * ig)); }

// R̂ of one voxel: three units, the indicators telescope to
// S = ς(z_top − z) − ς(−z), so W_l = D_l / S.
__device__ __forceinline__ float rhat(const VoxArgs &a, float H0, float H1, float z) {
  const float s0 = sig(H0 - z, a.inv_gamma), s1 = sig(H1 - z, a.inv_gamma);
  const float sb = sig(-z, a.inv_gamma), st = sig(a.z_top - z, a.inv_gamma);
  return (a.rho_m * (s0 - sb) + a.rho_a * (s1 - s0) + a.rho_r * (st - s1)) / (st - sb);
}

// Deviance-centred Poisson term and its λ̂-derivative with the R29 floor:
// ℓ = C(ln λ̂ − ln C) − λ̂ + C = C (log1p δ − δ) with δ = λ̂/C − 1 (C > 0), −λ̂ (C = 0).
__device__ __forceinline__ float loglik(float lam, float lam0, float cnt, float tau, float &dl) {
  const float fl = tau * lam0;
  dl = 0.f;
  if (lam < fl) lam = fl;
  else dl = cnt / lam - 1.f;
  if (cnt > 0.f) {
    const float d = lam / cnt - 1.f;
    float t;
    if (fabsf(d) < 0.125f)   // log1p δ − δ by its series (truncation < 1e-9 relative)
      t = d * d * fmaf(d, fmaf(d, fmaf(d, fmaf(d, fmaf(d, fmaf(d, fmaf(d, 1.f / 9.f, -1.f / 8.f), 1.f / 7.f),
                                                                 -1.f / 6.f), 1.f / 5.f), -1.f / 4.f), 1.f / 3.f), -0.5f);
    else
      t = log1pf(d) - d;
    return cnt * t;
  }
  return -lam;
}

// ---- chain lanes ---------------------------------------------------------
// A group of W = 32·VEC chains: lane l holds chains g·W + 32u + l (u < VEC), so
// the heights / ∂ℓ/∂H of each u are the coalesced 32-chain lines of the tix
// layout, while ΔR and r store the VEC values of a lane contiguously
// ([g][voxel | ray][lane][u]) and one gather of a G entry is a VEC-wide
// vector load: VEC x fewer instructions per chain and entry.
__device__ __forceinline__ int chain_of(int g, int VEC, int u, int lane) { return g * 32 * VEC + 32 * u + lane; }

template <int VEC>
__device__ __forceinline__ void ldv(const char *p, float (&d)[VEC]) {
  if constexpr (VEC == 1) {
    d[0] = __ldg((const float *)p);
  } else if constexpr (VEC == 2) {
    const float2 v = __ldg((const float2 *)p);
    d[0] = v.x; d[1] = v.y;
  } else {
    const float4 v = __ldg((const float4 *)p);
    d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
  }
}

template <int VEC>
__device__ __forceinline__ void stv(float *p, const float (&d)[VEC]) {
  if constexpr (VEC == 1) *p = d[0];
  else if constexpr (VEC == 2) *(float2 *)p = make_float2(d[0], d[1]);
  else *(float4 *)p = make_float4(d[0], d[1], d[2], d[3]);
}

// Layers k whose ΔR_v or ∂R̂_v/∂H can exceed e^{-VX_ZC} (relative) for any chain
// c in [c0, c1): z_k within VX_ZC γ of [min(H0, H_ref,0), max(H1, H_ref,1)].
// Outside it both R̂(H) and R0 equal the unit density to within
// 4 ρ_max e^{-24} (the sigmoids saturate), so their G ΔR terms sum to
// < 1e-9 λ_p(R0), below fp32 resolution of λ̂, and are skipped.
__device__ __forceinline__ void vx_band(const VoxArgs &a, int c0, int c1, int lane, int &k_lo, int &k_hi) {
  float lo = 3.0e38f, hi = -3.0e38f;
  for (int c = c0 + lane; c < c1; c += 32) {
    const float4 b = a.band[c];
    lo = fminf(lo, b.x);
    hi = fmaxf(hi, b.w);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  lo = fminf(lo, a.href_lo) - a.zc;
  hi = fmaxf(hi, a.href_hi) + a.zc;
  k_lo = 0;
  k_hi = a.nz - 1;
  if (lo == lo && hi == hi) {   // NaN heights: no skipping
    k_lo = max(0, (int)floorf(lo / a.dz));
    k_hi = min(a.nz - 1, (int)fminf(ceilf(hi / a.dz), 1.0e9f));
  }
}

template <int VEC>
__global__ void __launch_bounds__(MT_THREADS) k_vx_rhat_cl(VoxArgs a) {
  const int lane = threadIdx.x & 31, node = blockIdx.x * VX_WARPS + (threadIdx.x >> 5), g = blockIdx.y + a.g0;
  if (node >= a.N) return;
  int k_lo, k_hi;   // only the layers V2 / V3 read (vx_band)
  vx_band(a, g * 32 * VEC, min(a.C, (g + 1) * 32 * VEC), lane, k_lo, k_hi);
  float H0[VEC], H1[VEC];
#pragma unroll
  for (int u = 0; u < VEC; u++) {
    const int c = chain_of(g, VEC, u, lane);
    H0[u] = c < a.C ? a.H[tix(c, 0, node, a.N)] : 0.f;
    H1[u] = c < a.C ? a.H[tix(c, 1, node, a.N)] : 0.f;
  }
  float *out = a.dR + (((size_t)g * a.ng + (size_t)node * a.nz) * 32 + lane) * VEC;
  const float *r0 = a.R0 + (size_t)node * a.nz;
  for (int k = k_lo; k <= k_hi; k++) {
    const float z = k * a.dz, rk = r0[k];
    float d[VEC];
#pragma unroll
    for (int u = 0; u < VEC; u++) d[u] = rhat(a, H0[u], H1[u], z) - rk;
    stv<VEC>(out + (size_t)k * 32 * VEC, d);
  }
}

// acc[u] += Σ_j val_j · src_lane[idx_j][u] over one CSR / CSC segment.  Each
// chunk of 32 entries is loaded coalesced; the entries kept (all, or the
// in-band ones for BAND) are compacted into a per-warp shared list as
// {byte offset, value} (ballot + popc), zero-padded to a multiple of 4, and
// read back two at a time by broadcast LDS.128.
template <int VEC, bool BAND>
__device__ __forceinline__ int gather_dot(const int2 *e, int64_t beg, int64_t end, const char *src_lane, int lane,
                                          int nz, int k_lo, int k_hi, int4 *buf, float (&acc)[VEC]) {
  int2 *b2 = reinterpret_cast<int2 *>(buf);
  int kept = 0;
  for (int64_t j0 = beg; j0 < end; j0 += 32) {
    const bool in = j0 + lane < end;
    const int2 my = in ? e[j0 + lane] : make_int2(0, 0);
    bool keep = in;
    if (BAND) {
      const int k = my.x % nz;
      keep = keep && k >= k_lo && k <= k_hi;
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    const int n = __popc(m), n4 = (n + 3) & ~3;
    kept += n;
    if (keep) b2[__popc(m & ((1u << lane) - 1u))] = make_int2((int)((unsigned)my.x * (128u * VEC)), my.y);
    if (lane >= n && lane < n4) b2[lane] = make_int2(0, 0);
    __syncwarp();
    for (int t = 0; t < n4; t += 4) {
      const int4 q0 = buf[t >> 1], q1 = buf[(t >> 1) + 1];
      float d0[VEC], d1[VEC], d2[VEC], d3[VEC];
      ldv<VEC>(src_lane + (unsigned)q0.x, d0);
      ldv<VEC>(src_lane + (unsigned)q0.z, d1);
      ldv<VEC>(src_lane + (unsigned)q1.x, d2);
      ldv<VEC>(src_lane + (unsigned)q1.z, d3);
#pragma unroll
      for (int u = 0; u < VEC; u++) {
        acc[u] = fmaf(__int_as_float(q0.y), d0[u], acc[u]);
        acc[u] = fmaf(__int_as_float(q0.w), d1[u], acc[u]);
        acc[u] = fmaf(__int_as_float(q1.y), d2[u], acc[u]);
        acc[u] = fmaf(__int_as_float(q1.w), d3[u], acc[u]);
      }
    }
    __syncwarp();
  }
  return kept;
}

// The sub-range of row p that can hold layers [k_lo, k_hi]: entries of a row
// are in path order and z grows along every ray (d_z > 0), so its layers are
// non-decreasing; the per-row bucket offsets bound the in-band run.
__device__ __forceinline__ void row_range(const VoxArgs &a, int64_t p, int k_lo, int k_hi, int64_t &beg, int64_t &end) {
  const int64_t b0 = a.rowptr[p], b1 = a.rowptr[p + 1];
  const uint4 q = a.kofs[p];
  const unsigned o[8] = {q.x & 0xffffu, q.x >> 16, q.y & 0xffffu, q.y >> 16,
                         q.z & 0xffffu, q.z >> 16, q.w & 0xffffu, q.w >> 16};
  const int lo = k_lo / a.kb, hi = k_hi / a.kb + 1;
  beg = b0 + o[lo];
  end = hi < 8 ? b0 + o[hi] : b1;
}

// Block-sum the per-lane log-likelihood partials and add them to ll[c].
template <int VEC>
__device__ __forceinline__ void flush_ll(const double (&mine)[VEC], int lane, int g, int C, macc *ll) {
  __shared__ double sh[VX_WARPS][VEC][32];
#pragma unroll
  for (int u = 0; u < VEC; u++) sh[threadIdx.x >> 5][u][lane] = mine[u];
  __syncthreads();
  if (threadIdx.x < 32 * VEC) {
    const int u = threadIdx.x >> 5, l = threadIdx.x & 31;
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < VX_WARPS; w++) s += sh[w][u][l];
    const int c = chain_of(g, VEC, u, l);
    if (c < C) atomicAdd(ll + c, q_lld(s));
  }
}

template <int VEC>
__global__ void __launch_bounds__(MT_THREADS, VX_MINB) k_vx_fwd_cl(VoxArgs a) {
  const int lane = threadIdx.x & 31, g = blockIdx.y + a.g0;
  const int64_t p0 = ((int64_t)blockIdx.x * VX_WARPS + (threadIdx.x >> 5)) * a.rpw;
  const char *src = (const char *)(a.dR + ((size_t)g * a.ng * 32 + lane) * VEC);
  float *rout = a.r + ((size_t)g * a.R * 32 + lane) * VEC;
  __shared__ int4 bufs[VX_WARPS][16];
  int k_lo, k_hi;
  vx_band(a, g * 32 * VEC, min(a.C, (g + 1) * 32 * VEC), lane, k_lo, k_hi);
  double mine[VEC];
#pragma unroll
  for (int u = 0; u < VEC; u++) mine[u] = 0.0;
  long long kept = 0;
  for (int m = 0; m < a.rpw; m++) {
    const int64_t p = p0 + m;
    if (p >= a.R) break;
    float acc[VEC];
#pragma unroll
    for (int u = 0; u < VEC; u++) acc[u] = 0.f;
    int64_t beg, end;
    row_range(a, p, k_lo, k_hi, beg, end);
    kept += gather_dot<VEC, true>(a.csr, beg, end, src, lane, a.nz, k_lo, k_hi,
                          bufs[threadIdx.x >> 5], acc);
    const float2 lc = a.lc[p];
    float dl[VEC];
#pragma unroll
    for (int u = 0; u < VEC; u++) mine[u] += loglik(lc.x + acc[u], lc.x, lc.y, a.tau, dl[u]);
    stv<VEC>(rout + (size_t)p * 32 * VEC, dl);
  }
  if (a.gathered && lane == 0 && kept)
    atomicAdd(a.gathered, (unsigned long long)kept * 4ull * (unsigned long long)min(32 * VEC, a.C - g * 32 * VEC));
  flush_ll<VEC>(mine, lane, g, a.C, a.ll);
}

// Gᵀ pass: one warp per work item = a run of <= VX_CH consecutive CSC entries
// inside one node column (several light voxels, or a slice of a heavy one);
// ∂ℓ/∂H_l(node) += Σ_{v in item} (Σ_entries G_pv r_p) ∂R̂_v/∂H_l, float atomics.
__device__ __forceinline__ void vx_factors(const VoxArgs &a, float H0, float H1, int k, float &f0, float &f1) {
  const float z = k * a.dz;
  const float s0 = sig(H0 - z, a.inv_gamma), s1 = sig(H1 - z, a.inv_gamma);
  const float iS = a.inv_gamma / (sig(a.z_top - z, a.inv_gamma) - sig(-z, a.inv_gamma));
  f0 = s0 * (1.f - s0) * (a.rho_m - a.rho_a) * iS;
  f1 = s1 * (1.f - s1) * (a.rho_a - a.rho_r) * iS;
}

template <int VEC>
__global__ void __launch_bounds__(MT_THREADS, VX_MINB) k_vx_bwd_cl(VoxArgs a) {
  const int lane = threadIdx.x & 31, g = blockIdx.y + a.g0;
  const int64_t w = (int64_t)blockIdx.x * VX_WARPS + (threadIdx.x >> 5);
  __shared__ int4 bufs[VX_WARPS][16];
  if (w >= a.n_items) return;
  const VxItem it = a.items[w];
  float H0[VEC], H1[VEC], g0[VEC], g1[VEC];
#pragma unroll
  for (int u = 0; u < VEC; u++) {
    const int c = chain_of(g, VEC, u, lane);
    H0[u] = c < a.C ? a.H[tix(c, 0, it.node, a.N)] : 0.f;
    H1[u] = c < a.C ? a.H[tix(c, 1, it.node, a.N)] : 0.f;
    g0[u] = g1[u] = 0.f;
  }
  const char *src = (const char *)(a.r + ((size_t)g * a.R * 32 + lane) * VEC);
  int k_lo, k_hi;
  vx_band(a, g * 32 * VEC, min(a.C, (g + 1) * 32 * VEC), lane, k_lo, k_hi);
  int64_t pos = it.eb, v = (int64_t)it.node * a.nz + it.kb;
  for (int k = it.kb; pos < it.ee && k <= k_hi; k++, v++) {
    const int64_t cv = a.colptr[v + 1], vend = cv < (int64_t)it.ee ? cv : (int64_t)it.ee;
    if (vend <= pos) continue;
    if (k < k_lo) { pos = vend; continue; }
    float gR[VEC];   // (Gᵀ r)_v, this item's share
#pragma unroll
    for (int u = 0; u < VEC; u++) gR[u] = 0.f;
    gather_dot<VEC, false>(a.csc, pos, vend, src, lane, a.nz, 0, 0, bufs[threadIdx.x >> 5], gR);
#pragma unroll
    for (int u = 0; u < VEC; u++) {
      float f0, f1;
      vx_factors(a, H0[u], H1[u], k, f0, f1);
      g0[u] = fmaf(gR[u], f0, g0[u]);
      g1[u] = fmaf(gR[u], f1, g1[u]);
    }
    pos = vend;
  }
#pragma unroll
  for (int u = 0; u < VEC; u++) {
    const int c = chain_of(g, VEC, u, lane);
    if (c < a.C) {   // G is zero on entry (K3 clears what it reads)
      atomicAdd(a.G + tix(c, 0, it.node, a.N), q_g(g0[u]));
      atomicAdd(a.G + tix(c, 1, it.node, a.N), q_g(g1[u]));
    }
  }
}

// ---- row lanes (C < 16) ------------------------------------------------------
__global__ void __launch_bounds__(MT_THREADS) k_vx_rhat_rl(VoxArgs a) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)a.C * a.ng) return;
  const int c = (int)(t / a.ng);
  const int64_t v = t - (int64_t)c * a.ng;
  const int node = (int)(v / a.nz), k = (int)(v - (int64_t)node * a.nz);
  a.dR[t] = rhat(a, a.H[tix(c, 0, node, a.N)], a.H[tix(c, 1, node, a.N)], k * a.dz) - a.R0[v];
}


// Lane-partial Σ_j val_j · src[idx_j] over one segment (row lanes): four
// entries per lane per batch, all loads of a batch issued before any FMA.
__device__ __forceinline__ float seg_part_rl(const int2 *e, int64_t beg, int64_t end, const float *src, int lane) {
  float acc = 0.f;
  for (int64_t j0 = beg + lane; j0 < end; j0 += 128) {
    int2 x[4];
    float d[4];
#pragma unroll
    for (int u = 0; u < 4; u++) x[u] = j0 + 32 * u < end ? e[j0 + 32 * u] : make_int2(0, 0);
#pragma unroll
    for (int u = 0; u < 4; u++) d[u] = __ldg(src + x[u].x);
#pragma unroll
    for (int u = 0; u < 4; u++) acc = fmaf(__int_as_float(x[u].y), d[u], acc);
  }
  return acc;
}

// Row lanes: an 8-lane team per ray, four rays of a warp in flight; each lane
// gathers up to four in-band entries per batch, the team reduces by shuffles.
__global__ void __launch_bounds__(MT_THREADS) k_vx_fwd_rl(VoxArgs a) {
  __shared__ double sll[16];
  const int lane = threadIdx.x & 31, team = lane >> 3, tl = lane & 7;
  if (threadIdx.x < 16) sll[threadIdx.x] = 0.0;
  __syncthreads();
  const int64_t p0 = ((int64_t)blockIdx.x * VX_WARPS + (threadIdx.x >> 5)) * a.rpw;
  int k_lo, k_hi;
  vx_band(a, 0, a.C, lane, k_lo, k_hi);
  int kept = 0;
  for (int m = 0; m < a.rpw; m += 4) {
    const int64_t p = p0 + m + team;
    const bool live = m + team < a.rpw && p < a.R;
    int64_t beg = 0, end = 0;
    float2 lc = make_float2(1.f, 0.f);
    if (live) {
      row_range(a, p, k_lo, k_hi, beg, end);
      lc = a.lc[p];
    }
    for (int c = 0; c < a.C; c++) {
      const float *src = a.dR + (size_t)c * a.ng;
      float acc = 0.f;
      for (int64_t j0 = beg + tl; j0 < end; j0 += 32) {
        int2 x[4];
        float d[4];
#pragma unroll
        for (int u = 0; u < 4; u++) x[u] = j0 + 8 * u < end ? a.csr[j0 + 8 * u] : make_int2(0, 0);
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const int k = x[u].x % a.nz;
          const bool in = j0 + 8 * u < end && k >= k_lo && k <= k_hi;
          kept += in;
          d[u] = in ? __ldg(src + x[u].x) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 4; u++) acc = fmaf(__int_as_float(x[u].y), d[u], acc);
      }
      acc += __shfl_xor_sync(0xffffffffu, acc, 4);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      if (live && tl == 0) {
        float dl;
        const float l = loglik(lc.x + acc, lc.x, lc.y, a.tau, dl);
        a.r[(size_t)c * a.R + p] = dl;
        atomicAdd(&sll[c], (double)l);
      }
    }
  }
  if (a.gathered) {   // kept counts every chain's pass: 4 B per kept entry and chain
    const float tot = warp_allsum((float)kept);
    if (lane == 0 && tot > 0.f) atomicAdd(a.gathered, (unsigned long long)tot * 4ull);
  }
  __syncthreads();
  if (threadIdx.x < a.C) atomicAdd(a.ll + threadIdx.x, q_lld(sll[threadIdx.x]));
}

__global__ void __launch_bounds__(MT_THREADS) k_vx_bwd_rl(VoxArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (int64_t)blockIdx.x * VX_WARPS + (threadIdx.x >> 5);
  if (w >= a.n_items) return;
  const VxItem it = a.items[w];
  int k_lo, k_hi;
  vx_band(a, 0, a.C, lane, k_lo, k_hi);
  for (int c = 0; c < a.C; c++) {
    const float H0 = a.H[tix(c, 0, it.node, a.N)], H1 = a.H[tix(c, 1, it.node, a.N)];
    const float *r = a.r + (size_t)c * a.R;
    float g0 = 0.f, g1 = 0.f;
    int64_t pos = it.eb, v = (int64_t)it.node * a.nz + it.kb;
    for (int k = it.kb; pos < it.ee && k <= k_hi; k++, v++) {
      const int64_t cv = a.colptr[v + 1], vend = cv < (int64_t)it.ee ? cv : (int64_t)it.ee;
      if (vend <= pos) continue;
      if (k < k_lo) { pos = vend; continue; }
      const float acc = seg_part_rl(a.csc, pos, vend, r, lane);
      float f0, f1;
      vx_factors(a, H0, H1, k, f0, f1);
      g0 = fmaf(acc, f0, g0);
      g1 = fmaf(acc, f1, g1);
      pos = vend;
    }
    g0 = warp_allsum(g0);
    g1 = warp_allsum(g1);
    if (lane == 0) {
      atomicAdd(a.G + tix(c, 0, it.node, a.N), q_g(g0));
      atomicAdd(a.G + tix(c, 1, it.node, a.N), q_g(g1));
    }
  }
}

// ---- host: voxel walk of one ray (double) -----------------------------------
// Amanatides-Woo stepping over the column edges e_x, e_y (midpoints between
// nodes, clipped to the footprint) and the planes kΔz, from s = 0 to s_exit.
// Appends {voxel, length} for every piece of positive length.
struct Walker {
  int nx, ny, nz;
  double dz, z_top;
  std::vector<double> ex, ey;
  template <class F>
  void walk(double ox, double oy, double dx, double dy, double dzr, double s_exit, F &&emit) const {
    auto start = [](const std::vector<double> &e, int n, double o, double d) {
      int i = 0;
      for (int k = 1; k < n; k++)
        if (d < 0 ? e[k] < o : e[k] <= o) i = k;
      return i;
    };
    int i = start(ex, nx, ox, dx), j = start(ey, ny, oy, dy), k = 0;
    const double inf = INFINITY;
    auto tx_of = [&](int ii) {
      if (dx > 0) return ii + 1 < nx ? (ex[ii + 1] - ox) / dx : inf;
      if (dx < 0) return ii > 0 ? (ex[ii] - ox) / dx : inf;
      return inf;
    };
    auto ty_of = [&](int jj) {
      if (dy > 0) return jj + 1 < ny ? (ey[jj + 1] - oy) / dy : inf;
      if (dy < 0) return jj > 0 ? (ey[jj] - oy) / dy : inf;
      return inf;
    };
    auto tz_of = [&](int kk) { return kk + 1 < nz ? (kk + 1) * dz / dzr : inf; };
    double s = 0.0, tx = tx_of(i), ty = ty_of(j), tz = tz_of(k);
    for (;;) {
      double t = std::min(std::min(tx, ty), std::min(tz, s_exit));
      if (t > s) emit((int64_t)(i * ny + j) * nz + k, t - s);
      if (t >= s_exit) break;
      if (tx == t) { i += dx > 0 ? 1 : -1; tx = tx_of(i); }
      if (ty == t) { j += dy > 0 ? 1 : -1; ty = ty_of(j); }
      if (tz == t) { k += 1; tz = tz_of(k); }
      s = t;
    }
  }
};

template <class F>
void parallel_rays(int64_t R, F &&f) {
  unsigned T = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  std::vector<std::thread> th;
  for (unsigned t = 0; t < T; t++)
    th.emplace_back([&, t] {
      for (int64_t q = (int64_t)t; q < R; q += T) f(q);
    });
  for (auto &x : th) x.join();
}

}  // namespace

void voxel_free(mt_problem *p) {
  void *bufs[] = {p->vx.rowptr, p->vx.csr, p->vx.colptr, p->vx.csc, p->vx.lc, p->vx.R0, p->vx.dR, p->vx.r,
                  p->vx.items, p->vx.gathered, p->vx.kofs};
  for (void *b : bufs)
    if (b) cudaFree(b);
  p->vx = VoxelState{};
}

cudaError_t voxel_setup(mt_problem *p, int nz, float gamma, float tau, const float *Href) {
  voxel_free(p);
  if (nz == 0) return cudaSuccess;
  const int nx = p->nx, ny = p->ny, N = p->N;
  const int64_t R = p->R, ng = (int64_t)N * nz;
  Walker w;
  w.nx = nx; w.ny = ny; w.nz = nz;
  w.z_top = p->z_top;
  w.dz = (double)p->z_top / nz;
  w.ex.resize(nx + 1);
  w.ey.resize(ny + 1);
  for (int i = 0; i <= nx; i++)
    w.ex[i] = i == 0 ? p->hX[0] : (i == nx ? p->hX[nx - 1] : 0.5 * ((double)p->hX[i - 1] + p->hX[i]));
  for (int j = 0; j <= ny; j++)
    w.ey[j] = j == 0 ? p->hY[0] : (j == ny ? p->hY[ny - 1] : 0.5 * ((double)p->hY[j - 1] + p->hY[j]));
  // R0 = R̂(H_ref) in double (R28)
  const double rho[3] = {p->rho[0], p->rho[1], p->rho[2]};
  std::vector<double> R0(ng);
  auto sg = [&](double u) { return 1.0 / (1.0 + exp(-u / (double)gamma)); };
  for (int node = 0; node < N; node++)
    for (int k = 0; k < nz; k++) {
      double z = k * w.dz, b[4] = {0.0, Href[node], Href[N + node], (double)p->z_top}, D[3], S = 0, Rv = 0;
      for (int l = 0; l < 3; l++) { D[l] = sg(b[l + 1] - z) - sg(b[l] - z); S += D[l]; }
      for (int l = 0; l < 3; l++) Rv += D[l] / S * rho[l];
      R0[(size_t)node * nz + k] = Rv;
    }
  // per-ray geometry in double from the fp32 inputs
  auto ray = [&](int64_t q, double &ox, double &oy, double &dx, double &dy, double &dzr, double &s_exit,
                 double &L_ext) {
    const float4 A = p->h_ra[q], B = p->h_rb[q];
    ox = A.x; oy = A.y; dx = A.z; dy = A.w; dzr = B.x;
    double s_top = (double)p->z_top / dzr, s = s_top;
    if (dx > 0) s = fmin(s, ((double)p->hX[nx - 1] - ox) / dx);
    if (dx < 0) s = fmin(s, ((double)p->hX[0] - ox) / dx);
    if (dy > 0) s = fmin(s, ((double)p->hY[ny - 1] - oy) / dy);
    if (dy < 0) s = fmin(s, ((double)p->hY[0] - oy) / dy);
    s_exit = s;
    L_ext = s_top - s;
  };
  // pass 1: pieces per ray
  std::vector<int64_t> rowptr(R + 1, 0);
  parallel_rays(R, [&](int64_t q) {
    double ox, oy, dx, dy, dzr, se, le;
    ray(q, ox, oy, dx, dy, dzr, se, le);
    int64_t n = 0;
    w.walk(ox, oy, dx, dy, dzr, se, [&](int64_t, double) { n++; });
    rowptr[q + 1] = n;
  });
  for (int64_t q = 0; q < R; q++) rowptr[q + 1] += rowptr[q];
  const int64_t nnz = rowptr[R];
  // pass 2: G rows and λ_p(R0) (G_pv = −λ_p(R0) L_pv / Λ)
  std::vector<int2> csr(nnz > 0 ? nnz : 1);
  std::vector<float2> lc(R > 0 ? R : 1);
  const double Lam = p->att_len;
  parallel_rays(R, [&](int64_t q) {
    double ox, oy, dx, dy, dzr, se, le;
    ray(q, ox, oy, dx, dy, dzr, se, le);
    int64_t j = rowptr[q];
    std::vector<double> L;
    double O = 0.0;
    w.walk(ox, oy, dx, dy, dzr, se, [&](int64_t v, double l) {
      csr[j++].x = (int)v;
      L.push_back(l);
      O += l * R0[v];
    });
    O += p->rho[3] * le;
    const double lam0 = (double)p->h_w[q] * exp(-O / Lam);
    for (size_t m = 0; m < L.size(); m++) { float g = (float)(-lam0 * L[m] / Lam); memcpy(&csr[rowptr[q] + m].y, &g, 4); }
    lc[q] = make_float2((float)lam0, p->h_rb[q].w);
  });
  // per-row layer-bucket offsets (row_range)
  const int kb = (nz + 7) / 8;
  std::vector<uint4> kofs(R > 0 ? R : 1);
  for (int64_t q = 0; q < R; q++) {
    unsigned o[8];
    int64_t j = rowptr[q];
    for (int b = 0; b < 8; b++) {
      while (j < rowptr[q + 1] && csr[j].x % nz < b * kb) j++;
      o[b] = (unsigned)(j - rowptr[q]);
    }
    kofs[q] = make_uint4(o[0] | o[1] << 16, o[2] | o[3] << 16, o[4] | o[5] << 16, o[6] | o[7] << 16);
  }
  // CSC by a counting pass; each column's entries in increasing ray order
  std::vector<int64_t> colptr(ng + 1, 0);
  for (int64_t j = 0; j < nnz; j++) colptr[csr[j].x + 1]++;
  for (int64_t v = 0; v < ng; v++) colptr[v + 1] += colptr[v];
  std::vector<int2> csc(nnz > 0 ? nnz : 1);
  {
    std::vector<int64_t> fill(colptr.begin(), colptr.end() - 1);
    for (int64_t q = 0; q < R; q++)
      for (int64_t j = rowptr[q]; j < rowptr[q + 1]; j++) csc[fill[csr[j].x]++] = make_int2((int)q, csr[j].y);
  }
  // Gᵀ work items: runs of <= VX_CH entries inside one node column
  std::vector<VxItem> items;
  int ch = VX_CH;
  if (const char *ev = getenv("MT_VX_CH")) ch = std::max(32, atoi(ev));
  for (int node = 0; node < N; node++) {
    int64_t e0 = colptr[(int64_t)node * nz], e1 = colptr[(int64_t)(node + 1) * nz];
    int k = 0;
    for (int64_t e = e0; e < e1;) {
      while (colptr[(int64_t)node * nz + k + 1] <= e) k++;
      const int64_t ee = std::min<int64_t>(e + ch, e1);
      items.push_back(VxItem{node, k, e, ee});
      e = ee;
    }
  }
  std::vector<float> R0f(ng);
  for (int64_t v = 0; v < ng; v++) R0f[v] = (float)R0[v];
  // device
  VoxelState &s = p->vx;
  s.nz = nz; s.gamma = gamma; s.tau = tau; s.nnz = nnz; s.ng = ng;
  s.rpw_cl = VX_RPW_CL;
  s.vec = 0;
  s.gchunk = 0;
  if (const char *ev = getenv("MT_VX_GCHUNK")) s.gchunk = atoi(ev);
  if (const char *ev = getenv("MT_VX_VEC")) s.vec = atoi(ev) >= 4 ? 4 : (atoi(ev) >= 2 ? 2 : 1);
  s.rpw_rl = VX_RPW_RL;
  if (const char *ev = getenv("MT_VX_RPW")) s.rpw_cl = s.rpw_rl = std::max(1, atoi(ev));
  s.href_lo = *std::min_element(Href, Href + N);
  s.href_hi = *std::max_element(Href + N, Href + 2 * N);
  const size_t MC32 = (size_t)(p->max_chains > 0 ? (p->max_chains + 127) / 128 * 128 : 128);   // whole groups of up to 128
  cudaError_t e = cudaSuccess;
#define VALLOC(ptr, bytes) \
  if (e == cudaSuccess) e = cudaMalloc((void **)&(ptr), (bytes));
  VALLOC(s.rowptr, sizeof(int64_t) * (R + 1));
  VALLOC(s.csr, sizeof(int2) * csr.size());
  VALLOC(s.colptr, sizeof(int64_t) * (ng + 1));
  VALLOC(s.csc, sizeof(int2) * csc.size());
  VALLOC(s.lc, sizeof(float2) * lc.size());
  VALLOC(s.R0, sizeof(float) * ng);
  VALLOC(s.kofs, sizeof(uint4) * kofs.size());
  VALLOC(s.items, sizeof(VxItem) * std::max<size_t>(1, items.size()));
  VALLOC(s.gathered, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(s.gathered, 0, sizeof(unsigned long long));
  VALLOC(s.dR, sizeof(float) * MC32 * ng);
  VALLOC(s.r, sizeof(float) * MC32 * (size_t)(R > 0 ? R : 1));
#undef VALLOC
  if (e == cudaSuccess) e = cudaMemcpy(s.rowptr, rowptr.data(), sizeof(int64_t) * (R + 1), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(s.csr, csr.data(), sizeof(int2) * csr.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(s.colptr, colptr.data(), sizeof(int64_t) * (ng + 1), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(s.csc, csc.data(), sizeof(int2) * csc.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(s.lc, lc.data(), sizeof(float2) * lc.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(s.R0, R0f.data(), sizeof(float) * ng, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(s.kofs, kofs.data(), sizeof(uint4) * kofs.size(), cudaMemcpyHostToDevice);
  s.kb = kb;
  if (e == cudaSuccess && !items.empty())
    e = cudaMemcpy(s.items, items.data(), sizeof(VxItem) * items.size(), cudaMemcpyHostToDevice);
  s.n_items = (int64_t)items.size();
  if (e != cudaSuccess) voxel_free(p);
  return e;
}

cudaError_t launch_voxel(mt_problem *p, int C, const float *H, const float4 *band, macc *G, macc *ll,
                         cudaStream_t s) {
  const VoxelState &v = p->vx;
  VoxArgs a;
  a.C = C; a.N = p->N; a.ny = p->ny; a.nz = v.nz;
  a.R = p->R; a.ng = v.ng;
  a.dz = p->z_top / v.nz;
  a.inv_gamma = 1.f / v.gamma;
  a.z_top = p->z_top;
  a.tau = v.tau;
  a.rho_m = p->rho[0]; a.rho_a = p->rho[1]; a.rho_r = p->rho[2];
  a.H = H; a.R0 = v.R0; a.dR = v.dR; a.r = v.r;
  a.kofs = v.kofs; a.kb = v.kb;
  a.rowptr = v.rowptr; a.csr = v.csr; a.colptr = v.colptr; a.csc = v.csc; a.lc = v.lc;
  a.G = G; a.ll = ll;
  a.items = v.items; a.n_items = v.n_items;
  a.band = band;
  a.href_lo = v.href_lo; a.href_hi = v.href_hi;
  a.zc = VX_ZC * v.gamma;
  a.gathered = p->timing ? v.gathered : nullptr;
  a.g0 = 0;
  const bool rec = p->timing && p->n_rec < (int)p->ev_a.size();
  const unsigned nb_nodes = (unsigned)((p->N + VX_WARPS - 1) / VX_WARPS);
  const unsigned nb_bwd = (unsigned)std::max<int64_t>(1, (v.n_items + VX_WARPS - 1) / VX_WARPS);
  if (rec) cudaEventRecord(p->ev_a[p->n_rec], s);
  if (C >= 16) {
    // chains per lane: 4 once the 128-chain groups are mostly full (MT_VX_VEC overrides)
    const int vec = p->vx.vec > 0 ? p->vx.vec : (C >= 96 ? 4 : (C >= 48 ? 2 : 1));
    const unsigned groups = (unsigned)((C + 32 * vec - 1) / (32 * vec));
    a.rpw = p->vx.rpw_cl;
    const int64_t rpb = (int64_t)VX_WARPS * a.rpw;
    const unsigned nb_rays = (unsigned)((p->R + rpb - 1) / rpb);
    // group chunks: V1-V3 of `gc` groups back to back, so a chunk's ΔR and r are
    // still in L2 when V2 / V3 read them (gc = 0: all groups in one launch each)
    const int gc = p->vx.gchunk > 0 ? p->vx.gchunk : (int)groups;
#define VX_LAUNCH_CL(V)                                                                         \
    for (int g0 = 0; g0 < (int)groups; g0 += gc) {                                              \
      const unsigned ng_ = (unsigned)std::min(gc, (int)groups - g0);                            \
      a.g0 = g0;                                                                                \
      k_vx_rhat_cl<V><<<dim3(nb_nodes, ng_), MT_THREADS, 0, s>>>(a);                            \
      if (p->R > 0) k_vx_fwd_cl<V><<<dim3(nb_rays, ng_), MT_THREADS, 0, s>>>(a);               \
      k_vx_bwd_cl<V><<<dim3(nb_bwd, ng_), MT_THREADS, 0, s>>>(a);                               \
      p->all_launches += 3;                                                                     \
    }                                                                                           \
    if (rec) cudaEventRecord(p->ev_m[p->n_rec], s);
    if (vec == 4) { VX_LAUNCH_CL(4) } else if (vec == 2) { VX_LAUNCH_CL(2) } else { VX_LAUNCH_CL(1) }
#undef VX_LAUNCH_CL
  } else {
    const int64_t n = (int64_t)C * v.ng;
    k_vx_rhat_rl<<<(unsigned)((n + MT_THREADS - 1) / MT_THREADS), MT_THREADS, 0, s>>>(a);
    a.rpw = p->vx.rpw_rl;
    const int64_t rpb = (int64_t)VX_WARPS * a.rpw;
    if (p->R > 0) k_vx_fwd_rl<<<(unsigned)((p->R + rpb - 1) / rpb), MT_THREADS, 0, s>>>(a);
    if (rec) cudaEventRecord(p->ev_m[p->n_rec], s);
    k_vx_bwd_rl<<<nb_bwd, MT_THREADS, 0, s>>>(a);
    p->all_launches += 3;
  }
  if (rec) { cudaEventRecord(p->ev_b[p->n_rec], s); p->n_rec++; }
  p->trace_launches++;
  p->pairs += (double)C * (double)p->R;
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Measured roofline denominator of the voxel kernels: L2-resident gather
// bandwidth.  Each warp reads 512-B rows (a float4 per lane, the VEC = 4
// access of V2/V3) at hashed row indices of a `bytes`-sized buffer that fits
// in L2, all loads of a batch of 8 issued before use.
// ---------------------------------------------------------------------------
namespace {
__global__ void __launch_bounds__(MT_THREADS) k_l2_gather(const float4 *buf, unsigned rows, int iters, float *out) {
  const int lane = threadIdx.x & 31;
  unsigned h = (blockIdx.x * VX_WARPS + (threadIdx.x >> 5)) * 2654435761u + 12345u;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int i = 0; i < iters; i++) {
    float4 d[8];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      h = h * 1664525u + 1013904223u;
      d[u] = __ldg(buf + (size_t)(h % rows) * 32 + lane);
    }
#pragma unroll
    for (int u = 0; u < 8; u++) { acc.x += d[u].x; acc.y += d[u].y; acc.z += d[u].z; acc.w += d[u].w; }
  }
  if (acc.x + acc.y + acc.z + acc.w == 1.2345f) out[0] = acc.x;   // keep the loads
}
}  // namespace

cudaError_t run_l2_gather_peak(int device, size_t bytes, double *gbs) {
  cudaDeviceProp prop;
  cudaError_t e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) return e;
  float4 *buf = nullptr;
  float *out = nullptr;
  if ((e = cudaMalloc(&buf, bytes)) != cudaSuccess) return e;
  if ((e = cudaMalloc(&out, sizeof(float))) != cudaSuccess) { cudaFree(buf); return e; }
  cudaMemset(buf, 0, bytes);
  const unsigned rows = (unsigned)(bytes / 512);
  const int blocks = prop.multiProcessorCount * 8, iters = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_l2_gather<<<blocks, MT_THREADS>>>(buf, rows, 16, out);   // warm-up (brings the buffer into L2)
  double best = 0;
  for (int rep = 0; rep < 10; rep++) {
    cudaEventRecord(e0);
    k_l2_gather<<<blocks, MT_THREADS>>>(buf, rows, iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double b = 512.0 * 8.0 * iters * (double)blocks * VX_WARPS;
    best = std::max(best, b / (ms * 1e-3) / 1e9);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(buf);
  cudaFree(out);
  *gbs = best;
  return cudaGetLastError();
}
