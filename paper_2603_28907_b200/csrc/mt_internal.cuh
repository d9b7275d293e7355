// mt_internal.cuh — internal types of libmt (B200 / sm_100a).  Not part of the
// C ABI; never included by oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/mt.h"

#define MT_MAX_AXIS 128
#define MT_MAX_NODES 4096
#define MT_THREADS 256

// Fixed-point accumulators (R30).  ∂ℓ/∂H and the log-likelihood are
// summed as two's-complement int64 with RED.ADD.64: integer adds commute
// exactly, so every chain's result is bit-identical for any launch shape,
// order of processing (deferred pairs, dynamic ray queues), chain sharding over
// GPUs and, all-reduced as integers, ray sharding.
typedef unsigned long long macc;
#define MT_GQ 262144.0       // 2^18 units per 1 of ∂ℓ/∂H (range ±3.5e13, resolution 3.8e-6)
#define MT_LQ 16777216.0     // 2^24 units per 1 of ℓ (range ±5.5e11, resolution 6e-8)
__device__ __forceinline__ macc q_ll(float v) { return (macc)__float2ll_rn(v * (float)MT_LQ); }
__device__ __forceinline__ macc q_lld(double v) { return (macc)__double2ll_rn(v * MT_LQ); }
__device__ __forceinline__ macc q_raw(float v) { return (macc)__float2ll_rn(v); }   // v pre-scaled by MT_GQ
// Round-to-nearest of |v| < 2^22 to an integer on the FMA/ALU pipes (the magic-number
// trick: v + 1.5·2^23 puts round(v) in the low mantissa bits); F2I.S64 runs on the
// quarter-rate conversion unit, which the trace's scatter would otherwise saturate.
#define MT_QSMALL 4194304.0f
__device__ __forceinline__ macc q_small(float v) {
  return (macc)(long long)(__float_as_int(v + 12582912.0f) - 0x4B400000);
}
__device__ __forceinline__ macc q_g(float v) { return (macc)__float2ll_rn(v * (float)MT_GQ); }
__device__ __forceinline__ double dq_g(macc v) { return (double)(long long)v * (1.0 / MT_GQ); }
__device__ __forceinline__ double dq_ll(macc v) { return (double)(long long)v * (1.0 / MT_LQ); }

// Index of node k of surface l of chain c in the chain-interleaved layout
// [group = c/32][l][node][c % 32] used for the heights and ∂ℓ/∂H workspaces
// (a warp of 32 chains reads one 128-B line per node).
__host__ __device__ __forceinline__ size_t tix(int c, int l, int k, int N) {
  return ((size_t)(c >> 5) * 2 * N + (size_t)l * N + k) * 32 + (c & 31);
}

// Stored traversal cell word: the node offset (i n_y + j)·32 of the cell's
// (i, j) corner in the chain-interleaved layout (bits 0-16; N <= 4096), i
// (bits 17-23) and j (bits 24-30); MT_MAX_AXIS = 128.
__host__ __device__ __forceinline__ int cell_pack(int i, int j, int ny) {
  return ((i * ny + j) << 5) | (i << 17) | (j << 24);
}
__host__ __device__ __forceinline__ unsigned cell_off32(int w) { return (unsigned)w & 0x1ffffu; }
__host__ __device__ __forceinline__ int cell_i(int w) { return (w >> 17) & 127; }
__host__ __device__ __forceinline__ int cell_j(int w) { return (w >> 24) & 127; }

// Per-problem constants every trace launch needs (passed by value).
struct TraceConsts {
  int nx, ny, N;     // nodes per axis, nodes per surface
  float z_top;
  float k0, k1;      // ∂O/∂B0 = ρ_muck - ρ_air, ∂O/∂B1 = ρ_air - ρ_rock
  float inv_att;     // 1/Λ
};

// Ray SoA, one entry per ray of the shard:
//   a = {o_x, o_y, d_x, d_y}
//   b = {d_z, s_exit, t_base, C}
// with t_base = ln w - [C > 0] ln C - (ρ_rock s_exit + ρ_ext L_ext)/Λ, so that
// t = t_base - (k0 B0 + k1 B1)/Λ = ln(λ/C) (C > 0) or ln λ (C = 0).
struct TraceArgs {
  TraceConsts tc;
  const float *X, *Y;           // node coordinates
  const float4 *ray_a, *ray_b;
  const float *obase;           // ρ_rock s_exit + ρ_ext L_ext (path-length export only)
  const int32_t *trav_off;      // [R+1] CSR offsets of each ray's stored traversal
  const int2 *trav;             // {cell_pack(i, j), s_out bits} per cell, in ray order (a2)
  const float4 *trav_geo;       // per cell {u, v, α, β} at its entry (cell-local coordinates, a0)
  const float2 *trav_km;        // per cell {K = u β + v α, M = α β}: the ray-only parts of the solve's g1, g2
  // ray-lane traversal replay (k_trace_rl): per ray {n | i0 << 8 | j0 << 15, overflow word},
  // 2-bit exit codes of its cells (0 top, 1 x-line, 2 y-line, 3 vertex) for cells 0..63
  // and the code words of cells >= 64; the exit parameters are recomputed bit-exactly
  const int2 *rl_head;
  const uint4 *rl_code;
  const uint32_t *rl_ovf;
  const int32_t *perm;          // internal ray index -> caller's ray index
  int64_t R;                    // rays in the shard
  int64_t rays_per_block;
  int C;                        // chains in this call
  const float *H;               // [C][2][N] heights
  const void *cl;               // chain lanes, per evaluation: paired heights (k_cell_prep: float2
                                //   [group32][l][node][32]; k_cell_prep2: float4 [group64][l][node][32])
  const float *Hlo;             // fp32 residuals of the fp64 heights (0 for caller heights): the
                                //   fp64 re-solves of ill-conditioned cells use H + Hlo (HP2)
  const float4 *band;           // [C] (min H0, max H0, min H1, max H1)
  macc *G;                      // [C][2][N] ∂ℓ/∂H accumulator (fixed point MT_GQ, atomic adds)
  macc *ll;                     // [C] deviance-centred log-likelihood accumulator (fixed point MT_LQ)
  float *Lout, *Oout;           // path-length export: [C][R][3], [C][R]
  float4 *ovf_q;                // chain lanes: deferred pairs {c, ray, s_lo, s_hi} (an ill-
  int *ovf_n, *ovf_done;        //   conditioned cell or > RCAP crossings), done by k_trace_defer
  unsigned long long *ovf_total;   // cumulative deferred pairs
  int ovf_cap;
  unsigned *redo;               // [ceil(C R / 32)] pairs deferred after the queue filled
  unsigned long long *task_cost; // ray lanes, measurement only (mt_ray_cost): cycles per 32-ray task
};

enum { TRACE_LL = 0, TRACE_PATH = 1 };

struct FinishArgs {
  int nx, ny, N, P, C;
  float z_top;
  double inv_sigma[2];
  float car_r[2];
  double prior_const;           // Σ_l (1/2 ln det Q_l - N/2 ln 2π)
  int prior_on;
  const macc *G;                // ∂ℓ/∂H [C][2N], fixed point MT_GQ (zeroed after use)
  macc *ll;                     // [C] log-likelihood, fixed point MT_LQ (zeroed after use)
  float *x;                     // [C][P]
  const float *xin;             // [C][P] x to read (group-tiled K3: the leapfrog ping-pongs x between the
                                // caller's block and d_xalt so no tile reads a neighbour's updated x)
  float *grad;                  // [C][P]
  double *logp;                 // [C]
  int32_t *status;              // [C] or null
  float *mom;                   // [C][P] leapfrog momenta
  const float *eps;             // [C]
  float *H;                     // [C][2N] heights of the updated x (leapfrog)
  float *Hlo;                   // their fp32 residuals (H + Hlo = fp64 heights)
  float4 *band;                 // [C]
  float *kin;                   // [C] 1/2 |p|^2 after the last half kick
  int sample_r;                 // f2: state (x_0, x_1, ρ_0, ρ_1), r_l = logistic(ρ_l)
  const double *cs;             // [N] c_ab = 2(cos 2πa/n_x + cos 2πb/n_y) (torus spectrum)
  int ncp;                      // f2 non-centred: state (z_0, z_1, ρ_0, ρ_1), x = U(r) z
  double *xw;                   // [C][2N] fp64 x = U z of the current state (ncp)
  const float *minv;            // [P] diagonal inverse mass (null: identity)
};

enum { FIN_PLAIN = 0, FIN_STEP = 1, FIN_LAST = 2 };

// batched NUTS (kernels.cu, f1): per-chain tree state and workspace views
#define MT_NUTS_MAX_DEPTH 10
struct NutsChain {
  double H0, logW, logWs, lpL, lpR, lpw, lps, acc_sum;
  int dir, active, sub_ok, depth, n_leaf, diverging;
};
struct NutsArgs {
  float *thL, *pL, *gL, *thR, *pR, *gR;   // tree edges
  float *thw, *pw, *gw;                   // working state (the leaf being built)
  float *ths, *gs;                        // subtree proposal
  float *rho, *rhos, *tmp;                // momentum sums of the tree / subtree
  float *rck, *rsck;                      // U-turn checkpoints [depth][C][P]
  double *lpw_out;                        // logp of the working state (K3 output)
  NutsChain *st;
  int *any_active, *any_sub;
  const float *minv;                      // [P] diagonal inverse mass (null: identity)
};

struct VxItem { int node, kb; long long eb, ee; };   // Gᵀ work item (voxel.cu)

// f3 voxel / linearised model state (voxel.cu); nz == 0: the exact model is active
struct VoxelState {
  int nz = 0;
  float gamma = 1.f, tau = 1e-3f;
  int64_t nnz = 0, ng = 0;
  int64_t *rowptr = nullptr, *colptr = nullptr;
  int2 *csr = nullptr, *csc = nullptr;
  float2 *lc = nullptr;
  float *R0 = nullptr, *dR = nullptr, *r = nullptr;
  VxItem *items = nullptr;
  int64_t n_items = 0;
  float href_lo = 0, href_hi = 0;
  int rpw_cl = 4, rpw_rl = 16;   // rays per warp of V2 (MT_VX_RPW overrides)
  unsigned long long *gathered = nullptr;   // V2 gather-byte counter (while timing)
  uint4 *kofs = nullptr;         // per-row layer-bucket offsets
  int kb = 1;
  int gchunk = 0;                // chain groups per V1-V3 launch triple (0 = all; MT_VX_GCHUNK)
  int vec = 0;                   // chains per lane of the chain-lanes kernels (0 = by C; MT_VX_VEC)
};

struct mt_problem {
  int device = 0;
  int num_sms = 148;
  int nx = 0, ny = 0, N = 0, P = 0;
  int64_t R = 0, ray_lo = 0;
  int max_chains = 0;
  float z_top = 0;
  float car_r[2] = {0, 0};
  double sigma[2] = {0, 0}, logdetQ[2] = {0, 0};
  double loglik_offset = 0;
  float rho[4] = {0, 0, 0, 0};  // muck, air, rock, exterior
  float att_len = 0;
  std::vector<float> hX, hY, h_w;          // host copies for the voxel-model setup (internal ray order)
  std::vector<float4> h_ra, h_rb;
  VoxelState vx;
  int prior_on = 1;
  int sample_r = 0;             // f2: the CAR r_l are sampled (two more parameters per chain)
  double *d_cs = nullptr;       // [N] torus spectrum table (sample_r)
  int ncp = 0;                  // f2 non-centred parameterisation (implies sample_r)
  float *d_minv = nullptr;      // [P] diagonal inverse mass (null until mt_set_inverse_mass)
  uint64_t *d_iter = nullptr;   // device step counters (mt_set_step_counters, caller-owned): Philox
  int32_t *d_nprev = nullptr;   //   iteration of mt_hmc_step, Welford count of mt_stats_update
  float *d_xalt = nullptr;      // [max_chains][P] second x buffer of the group-tiled K3 leapfrog
  void *d_fin_part = nullptr;   // group-tiled K3 per-tile partials [groups][tiles][32] (FinPart, 48 B)
  unsigned *d_fin_ticket = nullptr;   // [groups] last-block tickets
  double *mb_red = nullptr;     // few-chain multi-block K3 scratch: [16][3] sums
  unsigned *mb_band = nullptr;  //   [16][4] band as float bits
  unsigned *mb_ticket = nullptr;   // [16] last-block tickets
  double *d_xw = nullptr;       // [max_chains][2N] fp64 x = U z (ncp)
  TraceConsts tc{};
  float *d_X = nullptr, *d_Y = nullptr;
  float4 *d_ray_a = nullptr, *d_ray_b = nullptr;
  float *d_obase = nullptr;
  int32_t *d_trav_off = nullptr;
  int32_t *d_perm = nullptr;
  std::vector<int32_t> perm, inv_perm;   // internal <-> caller ray order (host)
  int2 *d_trav = nullptr;
  float4 *d_trav_geo = nullptr;
  float2 *d_trav_km = nullptr;
  int2 *d_rl_head = nullptr;
  uint4 *d_rl_code = nullptr;
  uint32_t *d_rl_ovf = nullptr;
  float4 *d_ovf_q = nullptr;    // deferred-pair queue of the chain-lanes trace (see TraceArgs)
  int *d_ovf_n = nullptr;       // [4]: count, blocks done, 64-bit cumulative count
  int ovf_cap = 1 << 22;
  unsigned *d_redo = nullptr;   // (max_chains x R)-bit overflow bitmap of the deferred-pair queue
  int64_t trav_cells = 0;
  float *d_H = nullptr, *d_Hlo = nullptr;
  macc *d_G = nullptr;          // ∂ℓ/∂H accumulator, chain-interleaved, fixed point (R30)
  void *d_cl = nullptr;         // chain-lanes paired heights (TraceArgs::cl)
  float *d_Hc = nullptr;        // [min(max_chains, 16)][2N] contiguous heights for the ray-lanes trace
  float4 *d_band = nullptr;
  macc *d_ll = nullptr;         // log-likelihood accumulator, fixed point (R30)
  // HMC workspace
  float *d_x0 = nullptr, *d_g0 = nullptr, *d_mom = nullptr, *d_kin0 = nullptr, *d_kin1 = nullptr;
  double *d_lp0 = nullptr;
  // trace launch shape
  int trace_k = 0;              // chains per block (0 = auto)
  int trace_s = 0;              // ray splits (0 = auto)
  int cl_v = -1;                // chain-lanes kernel (MT_CL_V): -1 auto (c2 at C >= 64, else v0), 0 v0, 2 c2
  int chunk = 0;                // chain lanes: rays per block (a Morton-ordered chunk; 0 = by chain count)
  // batched NUTS workspace (allocated by the first mt_nuts_step)
  float *nuts_ws = nullptr;
  double *nuts_lp = nullptr;
  NutsChain *nuts_st = nullptr;
  int *nuts_flags = nullptr, *nuts_hflags = nullptr;
  float *nuts_rec_th = nullptr, *nuts_rec_g = nullptr;   // leaf record (mt_nuts_record)
  double *nuts_rec_lp = nullptr;
  int nuts_rec_max = 0;
  // in-library NCCL communicator (ray sharding; comm.cu)
  void *comm = nullptr;
  int comm_rank = 0, comm_world = 1;
  // measurement
  bool timing = false;
  std::vector<cudaEvent_t> ev_a, ev_b, ev_m;   // trace start, end, main-kernel end
  int n_rec = 0;
  double defer_ms = 0;
  int64_t trace_launches = 0, all_launches = 0;
  double pairs = 0;
};

// launchers (kernels.cu)
cudaError_t launch_heights(mt_problem *p, int C, const float *x, float *H, float4 *band,
                           cudaStream_t s);
cudaError_t launch_trace(mt_problem *p, int mode, int C, const float *H, const float4 *band,
                         macc *G, macc *ll, float *L, float *O, cudaStream_t s,
                         unsigned long long *task_cost = nullptr);
cudaError_t launch_finish(mt_problem *p, int mode, int C, float *x, float *grad, double *logp,
                          int32_t *status, float *mom, const float *eps, float *kin,
                          cudaStream_t s, const float *xin = nullptr);
bool use_mb(const mt_problem *p, int C);   // few chains: multi-block K3 and kicks, unfused leapfrog
bool use_fg(const mt_problem *p, int C);   // group-tiled K3 (the fused leapfrog ping-pongs x, d_xalt)
FinishArgs base_args(mt_problem *p, int C);   // per-problem constants of the per-chain kernels
// ncp.cu (f2 non-centred): heights of x = U z, K3, kick / drift (+ heights)
void launch_ncp_heights(mt_problem *p, const FinishArgs &a, int C, const float *x, cudaStream_t s);
void launch_ncp_finish(mt_problem *p, const FinishArgs &a, int C, cudaStream_t s);
void launch_ncp_kick(mt_problem *p, int mode, const FinishArgs &a, int C, cudaStream_t s);
cudaError_t launch_kick_drift(mt_problem *p, int C, float *x, float *mom, const float *grad,
                              const float *eps, cudaStream_t s);
cudaError_t launch_hmc_begin(mt_problem *p, int C, float *x, const double *logp,
                             const float *grad, const float *eps, uint64_t seed, uint64_t iter,
                             uint64_t chain_offset, cudaStream_t s);
cudaError_t launch_hmc_end(mt_problem *p, int C, float *x, double *logp, float *grad,
                           uint64_t seed, uint64_t iter, uint64_t chain_offset, float *acc_prob,
                           int32_t *accepted, int32_t *status, cudaStream_t s);
cudaError_t launch_momenta(mt_problem *p, int C, float *mom, uint64_t seed, uint64_t iter,
                           uint64_t chain_offset, cudaStream_t s);
cudaError_t build_traversal(mt_problem *p);
// voxel.cu (f3)
cudaError_t voxel_setup(mt_problem *p, int nz, float gamma, float tau, const float *Href);
void voxel_free(mt_problem *p);
cudaError_t launch_voxel(mt_problem *p, int C, const float *H, const float4 *band, macc *G, macc *ll,
                         cudaStream_t s);
cudaError_t launch_kick(mt_problem *p, int mode, int C, float *x, float *mom, const float *grad,
                        const float *eps, float *kin, cudaStream_t s);
enum { KICK_HALF_DRIFT = 0, KICK_FULL_DRIFT = 1, KICK_HALF_LAST = 2 };
cudaError_t run_nuts(mt_problem *p, int C, float *x, double *logp, float *grad, const float *eps, int max_depth,
                     uint64_t seed, uint64_t iter, uint64_t chain_offset, float *accept_stat, int32_t *depth,
                     int32_t *n_leaves, int32_t *status, cudaStream_t s, std::string &why);
// comm.cu
bool comm_unique_id(void *uid, std::string &why);
bool comm_attach(mt_problem *p, const void *uid, int rank, int world, std::string &why);
void comm_detach(mt_problem *p);
cudaError_t comm_allreduce_logp_grad(mt_problem *p, int C, double *logp, float *grad, cudaStream_t s,
                                     std::string &why);
cudaError_t launch_philox(const uint32_t *ctr, uint32_t k0, uint32_t k1, uint32_t *out,
                          int64_t n, int use_curand, cudaStream_t s);
cudaError_t run_fp32_peak(int device, double *tflops, double *mhz);
cudaError_t run_l2_gather_peak(int device, size_t bytes, double *gbs);
cudaError_t launch_stats(mt_problem *p, int C, const float *x, const float *acc, int32_t n_prev,
                         float *mean, float *m2, unsigned long long *acc_fixed, cudaStream_t s);
cudaError_t launch_tile(mt_problem *p, int C, const float *src, float *dst, int to_tiled,
                        cudaStream_t s);
cudaError_t launch_take_acc(mt_problem *p, int C, float *dldH, double *ll, cudaStream_t s);
cudaError_t launch_summary_finalize(mt_problem *p, int nz, const double *acc, double *out, cudaStream_t s);
cudaError_t launch_counter_add(uint64_t *iter, int32_t *nprev, cudaStream_t s);   // stats.cu
cudaError_t launch_summary(mt_problem *p, int C, const float *x, const double *logp, int nz, float gap,
                           double *acc, float *map_x, double *map_logp, cudaStream_t s);
cudaError_t launch_nested_rhat_partials(mt_problem *p, int C, int M, const float *mean, const float *m2,
                                        int32_t n, double *out, cudaStream_t s);
cudaError_t launch_rhat_partials(mt_problem *p, int C, const float *mean, const float *m2,
                                 int32_t n, double *out, cudaStream_t s);
