/*
 * mt.h — C ABI of the B200-native hot path of arXiv 2603.28907 ("Bayesian
 * muon tomography of block caves"): batched log-posterior + gradient over cave
 * geometries for many MCMC chains x many detector rays, and the fused HMC
 * leapfrog that consumes it.
 *
 * Citations: "P:a-b" = PAPER.md lines a-b (paper text, /root/reference at build
 * time); "R<k>" = reading k in DESIGN.md "Readings of the paper".
 *
 * CONVENTIONS (all entry points)
 *  - Return 0 (MT_OK) or a nonzero MT_E* code; mt_last_error() gives a
 *    thread-local message for the last nonzero return.
 *  - Ownership: mt_problem_create deep-copies every host array it is given;
 *    the caller may free them on return.  The problem owns its device buffers
 *    and workspace; mt_problem_destroy frees them.  State arrays (x, p, grad,
 *    logp, eps, status, accept_prob, accepted, H, dldH, L, O) are CALLER-OWNED
 *    DEVICE memory on the problem's device (e.g. torch CUDA tensors),
 *    C-contiguous; the library never frees them.
 *  - Layout of one chain's parameter block (P = 2*n_x*n_y floats): [l][ix][iy],
 *    iy fastest (right-most-fastest); l = 0 muck top (paper layer
 *    1), l = 1 cave back (paper layer 2) (R4).  A state block is
 *    [C][P].  Heights H and dldH use the same [C][2][n_x][n_y] layout, metres
 *    above the detector plane z = 0 (R5).
 *  - Streams: per-evaluation calls are asynchronous and stream-ordered on the
 *    given cudaStream_t (NULL = legacy default stream); there is no implicit
 *    device sync.  One stream at a time per problem (the workspace is not
 *    re-entrant).  mt_problem_create / destroy and mt_debug_traversal are
 *    synchronous.  Per-evaluation calls are CUDA-graph capturable.
 *  - Non-finite results are not an error return: per-chain status bits
 *    (1 = non-finite logp/grad, 2 = HMC divergence, rejected).
 */
#ifndef MT_H
#define MT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mt_problem mt_problem;
typedef struct CUstream_st *mt_stream; /* == cudaStream_t */

enum {
  MT_OK = 0,
  MT_EINVAL = 1, /* bad descriptor / argument (message says which) */
  MT_ENOMEM = 2, /* device or host allocation failed */
  MT_ECUDA = 3,  /* CUDA runtime error (message holds cudaGetErrorString) */
  MT_ENCCL = 4,  /* NCCL error in the in-library communicator (message holds ncclGetErrorString) */
  MT_ESTATE = 5  /* call not valid in the current state */
};

enum { MT_STATUS_NONFINITE = 1, MT_STATUS_DIVERGENT = 2 };

/* Problem description (all pointers are HOST memory, read during create).
 * Geometry (R2/R3): control nodes at (node_x[i], node_y[j]); the
 * surfaces are bilinear in each cell.  Coordinates must be multiples of
 * 2^-12 m with |v| < 2^11 m (exact traversal predicates, HP3).
 * Rays (R10/R11): one ray per pixel from detector ray_det[p] in unit
 * direction ray_dir[p] (d_z > 0); expected counts λ_p = ray_w[p]*exp(-O_p/att_len)
 * (R9) with opacity O_p = ∫ρ du through muck (z < H0), air
 * (H0 <= z < H1), rock (H1 <= z < z_top) inside the footprint and rho_ext
 * beyond a side exit up to z_top (R7).  Observed counts C_p ~ Poisson(λ_p)
 * (P:403-404).  Prior (R13/R14): x_l ~ N(0, Q_l^-1), Q_l = 4I - r_l A
 * on the periodic 4-neighbour grid, heights by the Gaussian copula
 * ǔ = Φ(x/σ_l) and stick-breaking H0 = ǔ0 z_top, H1 = H0 + ǔ1 (z_top - H0). */
typedef struct {
  int32_t n_x, n_y;          /* nodes per axis, >= 3, n_x*n_y <= 4096 */
  const float *node_x;       /* [n_x] strictly increasing */
  const float *node_y;       /* [n_y] strictly increasing */
  float z_top;               /* known flat top surface (m above z = 0) (R6) */
  float rho_muck, rho_air, rho_rock, rho_ext; /* g/cm^3, >= 0 (R8) */
  float att_len;             /* Λ > 0, g/cm^3*m (R9) */
  float car_r[2];            /* CAR r_l in [0, 1) */
  int32_t n_det;
  const float *det_xyz;      /* [n_det][3]; x,y strictly inside the footprint, z == 0 */
  int64_t n_rays;
  const int32_t *ray_det;    /* [n_rays] detector index */
  const float *ray_dir;      /* [n_rays][3] unit (|1-|d|| <= 1e-6), d_z > 0 */
  const float *ray_w;        /* [n_rays] exposure x solid angle x efficiency, > 0 */
  const int32_t *counts;     /* [n_rays] observed C_p >= 0 */
  int64_t ray_lo, ray_hi;    /* this rank's ray shard [ray_lo, ray_hi); (0, n_rays) unsharded */
  int32_t device;            /* CUDA device ordinal */
  int32_t max_chains;        /* capacity of the per-chain workspace */
  int32_t sample_r;          /* 0: r_l = car_r[l] fixed (R13, the hot path).  1: hierarchical r_l
                                (SURVEY §8(f) f2): each chain's state gains two
                                parameters ρ_0, ρ_1 with r_l = 1/(1+e^{-ρ_l}) ~ Unif(0,1); the
                                prior, σ_l and ln det Q_l then follow each chain's r_l (car_r unused) */
  int32_t noncentred;        /* 1 (requires sample_r): the paper's non-centred parameterisation
                                (R13d): the state is (z_0, z_1, ρ_0, ρ_1) with
                                z_l ~ N(0, I) and x_l = Q(r_l)^{-1/2} z_l (the symmetric root, applied
                                as a circulant by the 2-D DFT in fp64); logp = ll - ½|z|² - N ln 2π
                                + Σ ln r_l(1-r_l).  mt_nuts_step is not available in this mode. */
} mt_problem_desc;

/* Validate the description, precompute per-ray constants (in-box extent,
 * exterior rock length, deviance-centred log-weight) in double on the host,
 * upload them as an fp32 SoA, allocate the workspace.  Synchronous.
 * Errors: MT_EINVAL (message names the offending field), MT_ENOMEM, MT_ECUDA.
 *
 * Tuning environment variables, read here (performance only: results are
 * independent of them up to fp32 summation order; unset = the measured
 * defaults in DESIGN.md):
 *   MT_TRACE_K      1 = ray lanes, 32 = chain lanes (default: chain lanes iff C >= 16)
 *   MT_TRACE_S      trace grid splits over the rays
 *   MT_CHUNK        rays per chain-lanes block chunk (default 256 / 512)
 *   MT_OVF_CAP      deferred-pair queue capacity (tests force the bitmap overflow path)
 *   MT_RAY_ORDER    0 = input ray order instead of the Morton order
 *   MT_ORDER_Z      reference height of the Morton order, fraction of z_top
 *   MT_NO_MB        disable the few-chain multi-block K3 / kick kernels
 *   MT_VX_CH, MT_VX_GCHUNK, MT_VX_VEC, MT_VX_RPW   voxel model (mt_voxel_model)
 *                   work-item size, gather chunk, chains per lane, rows per warp */
int mt_problem_create(const mt_problem_desc *desc, mt_problem **out);

/* Free everything the problem owns.  NULL-safe.  Synchronous. */
int mt_problem_destroy(mt_problem *p);

/* P = 2*n_x*n_y (+ 2 with sample_r: ρ_0, ρ_1 last) parameters per chain; rays in this shard. */
int32_t mt_num_params(const mt_problem *p);
int64_t mt_num_rays(const mt_problem *p);

/* Σ_p (C_p ln C_p - C_p - ln Γ(C_p+1)) over this shard: add it to the
 * deviance-centred log-likelihood returned below to get the standard Poisson
 * log-likelihood Σ_p [C_p ln λ_p - λ_p - ln Γ(C_p+1)] (R15). */
double mt_loglik_offset(const mt_problem *p);

/* σ_l (marginal std of the torus CAR field, P:589-590 / R14) and ln det Q_l. */
int mt_prior_constants(const mt_problem *p, double sigma[2], double logdetQ[2]);

/* Unnormalised log-posterior and its gradient for C chains.
 *   x     [C][P] float  latent CAR fields (device)
 *   logp  [C]   double  Σ_p ℓ_p^dev + Σ_l log N(x_l; 0, Q_l^-1)   (device)
 *                       where ℓ_p^dev = C_p(ln λ_p - ln C_p) - λ_p + C_p (R15)
 *   grad  [C][P] float  ∂logp/∂x (device)
 *   status[C] int32 or NULL (device)
 * With a ray shard (ray_lo > 0 or ray_hi < n_rays) the likelihood part covers
 * the shard only and the prior is added on the shard with ray_lo == 0, so a
 * SUM over shards gives the full result.  Errors: MT_EINVAL (C < 0,
 * C > max_chains, NULL pointer), MT_ECUDA. */
int mt_logpost_grad(mt_problem *p, int32_t C, const float *x, double *logp, float *grad,
                    int32_t *status, mt_stream stream);

/* L velocity-Verlet (kick-drift-kick) steps with identity mass (P:625-642,
 * R19), per-chain step size eps[C] (device).  On entry logp/grad must hold the
 * values at x (e.g. from mt_logpost_grad); on return x, p, logp, grad are
 * advanced by L steps.  L >= 0. */
int mt_leapfrog(mt_problem *p, int32_t C, float *x, float *mom, double *logp, float *grad,
                const float *eps, int32_t L, mt_stream stream);

/* Momenta p ~ N(0, I) from Philox4x32-10: key = (seed lo, seed hi), counter =
 * (q, chain_offset + c, iter mod 2^32, 0) for parameters 4q..4q+3, uniforms
 * (k + 1/2) 2^-32, Box-Muller on word pairs (0,1), (2,3) (R22). */
int mt_draw_momenta(mt_problem *p, int32_t C, float *mom, uint64_t seed, uint64_t iter,
                    uint64_t chain_offset, mt_stream stream);

/* One HMC transition per chain: draw momenta as above, L leapfrog
 * steps, Hamiltonian H = -logp + |p|^2/2, accept iff ln u < -ΔH with u from
 * Philox counter (0, chain, iter, 1) word 0; divergent (ΔH > 1000 or
 * non-finite) proposals are rejected and flagged.  x/logp/grad are updated in
 * place (restored on reject).  accept_prob [C] float = min(1, exp(-ΔH));
 * accepted [C] int32; status [C] or NULL. */
int mt_hmc_step(mt_problem *p, int32_t C, float *x, double *logp, float *grad, const float *eps,
                int32_t L, uint64_t seed, uint64_t iter, uint64_t chain_offset, float *accept_prob,
                int32_t *accepted, int32_t *status, mt_stream stream);

/* ---- ray sharding over GPUs (BASELINE configs[4]) ---------
 * Rays are independent given a chain's heights, so a problem created with a
 * ray shard computes partial sums; with a communicator attached, every
 * per-evaluation call (mt_logpost_grad, and each of the L evaluations inside
 * mt_leapfrog / mt_hmc_step) all-reduces (SUM) the per-chain [logp, grad]
 * in-stream with NCCL over NVLink before the kick that consumes them, so all
 * ranks hold identical (replicated) chain states and trajectories.  The prior
 * term is added by the shard with ray_lo == 0 only.
 *
 * mt_comm_unique_id: an NCCL unique id (128 bytes, host) on one rank; the
 *   caller broadcasts it (e.g. torch.distributed.broadcast_object_list).
 * mt_attach_comm: every rank (one process per GPU, the problem's device)
 *   creates the communicator of `world` ranks from that id (collective,
 *   synchronous; NCCL is loaded from the already-loaded libnccl.so.2 of the
 *   process, else the system one).  Replaces any attached communicator.
 * mt_detach_comm: destroy it (also done by mt_problem_destroy).
 * Errors: MT_EINVAL, MT_ENCCL (NCCL missing or failing). */
int mt_comm_unique_id(void *uid128);
int mt_attach_comm(mt_problem *p, const void *uid128, int32_t rank, int32_t world);
int mt_detach_comm(mt_problem *p);

/* One No-U-Turn transition per chain (trajectory
 * capped at 2^max_depth leapfrog steps; reading R26 in DESIGN.md):
 * momenta as mt_draw_momenta; the trajectory doubles up to max_depth times in
 * Philox-drawn directions (counter (depth, chain, iter, 2)); leaves are chosen
 * by progressive multinomial sampling (counters (leaf, chain, iter, 3) and
 * (depth, chain, iter, 4)); subtrees stop on a U-turn of any aligned
 * sub-trajectory or a divergence (ΔH > 1000 / non-finite).  All chains advance
 * in lockstep, one leaf (one log-posterior+gradient evaluation of all C
 * chains) per step; finished chains idle.
 *   x, logp, grad (in/out): on entry the current state with its logp/grad, on
 *     return the selected state with its logp/grad;
 *   accept_stat [C] float: mean min(1, e^{-ΔH}) over the leaves (step-size
 *     adaptation); depth, n_leaves [C] int32 or NULL; status [C] or NULL
 *     (bit 2 = divergent trajectory).
 * 1 <= max_depth <= 10.  Synchronous (the doubling loop reads one flag per
 * depth), not graph-capturable; the first call allocates the tree workspace
 * ((16 + 20) x max_chains x P floats).  With a ray-shard communicator every
 * leaf is all-reduced like mt_leapfrog. */
int mt_nuts_step(mt_problem *p, int32_t C, float *x, double *logp, float *grad, const float *eps,
                 int32_t max_depth, uint64_t seed, uint64_t iter, uint64_t chain_offset, float *accept_stat,
                 int32_t *depth, int32_t *n_leaves, int32_t *status, mt_stream stream);

/* Debug / parity record of mt_nuts_step's leaves (f1; the depth-8 replay test):
 * while set, every leaf evaluation of the following mt_nuts_step calls stores the
 * leaf state of all C chains at leaf index k = 2^depth - 1 + t (evaluation order;
 * leaves skipped because every chain had stopped are not written): th [k][C][P]
 * float, g [k][C][P] float (its gradient), lp [k][C] double (its logp), for
 * k < max_leaves.  DEVICE buffers, caller-owned; th == NULL switches it off. */
int mt_nuts_record(mt_problem *p, float *th, float *g, double *lp, int32_t max_leaves);

/* Per-iteration sampler statistics (step-size adaptation and R-hat, P:652-653,
 * P:671-687; readings R20/R21).  Any of the three groups may be skipped by
 * passing NULL:
 *   accept_prob [C] + acc_fixed [2] (device uint64): acc_fixed[0] +=
 *     Σ_c round(accept_prob_c · 2^32), acc_fixed[1] += C — exact integer sums,
 *     so a cross-rank SUM is order-independent;
 *   x [C][P] + mean, m2 [C][P] (device fp32): Welford update with count
 *     n_prev + 1 (mean/m2 zero before the first sampling iteration). */
int mt_stats_update(mt_problem *p, int32_t C, const float *x, const float *accept_prob,
                    int32_t n_prev, float *mean, float *m2, uint64_t *acc_fixed, mt_stream stream);

/* R-hat partial sums over this rank's C chains after n Welford updates:
 * out [3][P] (device double) = (Σ_c mean_c, Σ_c mean_c², Σ_c m2_c/(n-1)).
 * A SUM over ranks gives the global between/within-chain statistics. */
int mt_rhat_partials(mt_problem *p, int32_t C, const float *mean, const float *m2, int32_t n,
                     double *out, mt_stream stream);

/* Nested R̂ partial sums (n_super super-chains of M chains that share
 * their start, Margossian et al.; reading R21b): chains [kM, (k+1)M) of this
 * rank form super-chain k (C % M == 0; super-chains never straddle ranks).
 * After n >= 1 Welford updates (n = 1: the paper's keep-last protocol), out
 * [3][P] (device double) = (Σ_k m_k, Σ_k m_k², Σ_k W_k) with m_k the
 * super-chain mean and W_k its pooled variance (mean within-chain variance +
 * variance of its chain means).  A SUM over ranks gives B = var_k m_k
 * (unbiased), W = mean_k W_k and nested R̂ = sqrt(1 + B/W) per parameter. */
int mt_nested_rhat_partials(mt_problem *p, int32_t C, int32_t M, const float *mean, const float *m2, int32_t n,
                            double *out, mt_stream stream);

/* Posterior summaries (reading R27), accumulated
 * over draws (call once per kept draw set, e.g. each sampling iteration, or once
 * with the last draws of the keep-last protocol):
 *   acc (device double, zeroed by the caller), size 1 + 3N + 6 N nz:
 *     [0] number of draws; [1, 1+2N) Σ heights (mean heights);
 *     [1+2N, 1+3N) #draws with air thickness H1 - H0 > gap (m);
 *     then Σ D and Σ D² of the smooth layer indicators D^(l) (l = muck, air,
 *     rock, γ = 1 m) on voxel columns at the nodes, z_k = k z_top/nz,
 *     laid out [sum|sum²][l][node][k] (indicator-std tomography).
 *   map_x [P] / map_logp [1] (device, optional, map_logp initialised to -inf):
 *     replaced by the highest-logp draw among x when higher (MAP).
 * Uses (and overwrites) the problem's height workspace. */
int mt_summary_update(mt_problem *p, int32_t C, const float *x, const double *logp, int32_t nz, float gap,
                      double *acc, float *map_x, double *map_logp, mt_stream stream);

/* Device-side step counters, for capturing a sampling step in a CUDA graph (a
 * captured launch keeps the host scalars it was captured with):
 *   iter    DEVICE uint64 [1] or NULL: mt_hmc_step then takes the Philox iteration
 *           (R22) from *iter instead of its `iter` argument, and adds 1 to *iter at
 *           the end of the step (in stream order);
 *   n_prev  DEVICE int32 [1] or NULL: mt_stats_update's Welford update then takes
 *           the count from *n_prev instead of its `n_prev` argument and adds 1.
 * Caller-owned; NULL restores the host arguments.  The results are those of the
 * host-argument calls with the same values (tests/test_gpu_graph.py).
 * Errors: MT_EINVAL (p NULL). */
int mt_set_step_counters(mt_problem *p, uint64_t *iter, int32_t *n_prev);

/* The summaries from the accumulators of mt_summary_update (R27):
 *   acc  DEVICE double, as filled by mt_summary_update (acc[0] >= 1 draws).
 *   out  DEVICE double [3N + 3 N nz], caller-owned:
 *        [0, 2N)        mean heights, [surface][node];
 *        [2N, 3N)       air-gap exceedance probability per node;
 *        [3N, 3N+3N nz) indicator std sqrt(max(E[D²] - E[D]², 0)), laid out
 *                       [unit l][node][layer k] (indicator-std tomography,
 *                       P:789-811).
 * Asynchronous on `stream`.  Errors: MT_EINVAL (NULL, nz < 1), MT_ECUDA. */
int mt_summary_finalize(mt_problem *p, int32_t nz, const double *acc, double *out, mt_stream stream);

/* Diagonal inverse mass matrix M^-1 for HMC and NUTS (NumPyro's default
 * adapted diagonal mass, the paper's sampler P:643-653; R19b):
 * momenta p ~ N(0, M), drift x += ε M^-1 p, kinetic energy ½ pᵀ M^-1 p, the
 * NUTS U-turn criterion on the velocities M^-1 p.  One vector shared by all
 * chains of the problem (the driver adapts it from pooled warm-up variances).
 *   minv   DEVICE [n] fp32, every entry finite and > 0; copied (synchronous).
 *          NULL restores the identity.
 *   n      must equal P (mt_num_params).
 * Affects mt_draw_momenta, mt_leapfrog, mt_hmc_step, mt_nuts_step.
 * Errors: MT_EINVAL (n, non-positive entries), MT_ENOMEM, MT_ECUDA. */
int mt_set_inverse_mass(mt_problem *p, const float *minv, int32_t n);

/* ---- the paper's voxel / sigmoid / linearised forward model (f3) -------- */

/* Switch the problem's likelihood to the paper's own approximate forward
 * model (readings R28/R29):
 *   voxel grid: column (i,j) at layer-grid node (i,j) between the midpoints of
 *     neighbouring nodes, n_z layers [kΔz, (k+1)Δz), Δz = z_top/n_z,
 *     v = (i n_y + j) n_z + k;
 *   R̂_v(H) = Σ_l W_v^(l) ρ_l, W = D/ΣD, D^(l) = ς_γ(H_l − kΔz) − ς_γ(H_{l−1} − kΔz)
 *     (P:344-383), three units muck/air/rock;
 *   λ̂(H) = λ(R0) + G (R̂(H) − R0), G = ∂λ/∂R at R0 = R̂(H_ref),
 *     floored at τ λ(R0) with zero derivative below (R29);
 *   ℓ = Σ_p C_p (ln λ̂_p − ln C_p) − λ̂_p + C_p (the exact model's deviance form).
 * After the call mt_logpost_grad, mt_leapfrog, mt_hmc_step, mt_nuts_step and
 * mt_loglik_heights evaluate this model (the prior, heights map, samplers and
 * communicator are unchanged); mt_path_lengths stays the exact tracer's.
 *   n_z      layers (1..4096); 0 switches back to the exact model and frees
 *            the voxel buffers (gamma, tau, H_ref ignored).
 *   gamma    sigmoid scale γ (> 0, metres; the paper's value is 1).
 *   tau      floor fraction τ in [0, 1) (R29; 1e-3 in the tests and bench).
 *   H_ref    HOST [2][n_x][n_y] fp32 reference geometry (muck top, cave back).
 * Setup builds G (CSR by ray and CSC by voxel, fp32 values) on the host in
 * double and uploads it: one synchronous call, O(nnz) host work and device
 * memory 16 B per non-zero + 4·(n_grid + R)·⌈max_chains/32⌉·32 B of
 * workspace.  Limits: n_x n_y n_z <= 2^23 voxels and <= 2^23 rays per shard.
 * Errors: MT_EINVAL (arguments, limits), MT_ENOMEM, MT_ECUDA; on error the
 * exact model is active. */
int mt_voxel_model(mt_problem *p, int32_t n_z, float gamma, float tau, const float *H_ref);

/* Active voxel model: n_z (0 = exact model), non-zeros of G, n_grid. */
int mt_voxel_info(const mt_problem *p, int32_t *n_z, int64_t *nnz, int64_t *n_grid);

/* Cumulative ΔR bytes the λ̂ kernel gathered while timing was on
 * (mt_timing_start .. mt_timing_read): 4 B per chain and in-band G entry, the
 * algorithmic gather traffic of the voxel model's roofline.
 * Synchronises the device. */
int mt_voxel_counters(mt_problem *p, uint64_t *gathered_bytes);

/* Measured roofline denominator for the voxel kernels: the best of 10 runs of
 * a gather kernel reading 512-B rows at hashed indices of an L2-resident
 * buffer of `bytes` (>= 1 MiB; 32 MiB in bench.py), in GB/s. */
int mt_measure_l2_gather(int32_t device, int64_t bytes, double *gbs);

/* ---- parity / debug entry points (not on the hot path) ---------------- */

/* Heights map of x (device [C][P] -> device H [C][2][n_x][n_y]). */
int mt_heights(mt_problem *p, int32_t C, const float *x, float *H, mt_stream stream);

/* Deviance-centred log-likelihood (device ll [C], double) and ∂ll/∂H (device
 * dldH [C][2][n_x][n_y]) for caller-given heights H (device, same layout):
 * the trace/adjoint path alone. */
int mt_loglik_heights(mt_problem *p, int32_t C, const float *H, double *ll, float *dldH,
                      mt_stream stream);

/* In-box path lengths per (chain, ray of this shard): L [C][R][3] = (muck,
 * air, rock) and opacity O [C][R] (device) for caller-given heights H. */
int mt_path_lengths(mt_problem *p, int32_t C, const float *H, float *L, float *O,
                    mt_stream stream);

/* Ordered cells (i, j) of ray `ray` (index within this shard), with s_in,
 * s_out; HOST outputs, up to cap entries, *n = number of cells.  Synchronous;
 * runs the same device traversal the trace kernel uses. */
int mt_debug_traversal(mt_problem *p, int64_t ray, int32_t *ij, float *s_in, float *s_out,
                       int32_t cap, int32_t *n);

/* Every ray's stored traversal (a2: the cells the trace kernels read, built
 * once per problem by the exact device DDA, P:234-235 / R16), in the caller's
 * ray order of this shard, as CSR with HOST outputs: with ij == NULL only
 * off [R+1] is written (off[q+1] - off[q] = cells of ray q); then ij
 * [off[R]][2] receives (i, j) and s_out [off[R]] each cell's exit parameter
 * (fp32, m).  Synchronous.  MT_EINVAL for a NULL problem or off. */
int mt_traversal_all(mt_problem *p, int64_t *off, int32_t *ij, float *s_out);

/* Trace work per ray of this shard for one chain state (ray-shard balancing,
 * SURVEY §8(e)): work[q] (HOST [R], caller's ray order) = the number of the
 * ray's stored cells whose z-range meets the chain's height band [min H0,
 * max H1] (the cells the trace walks), for the chain state x (DEVICE [P]).
 * Synchronous.  MT_EINVAL for NULL arguments. */
int mt_ray_work(mt_problem *p, const float *x, int32_t *work);

/* Measured trace cost per ray of this shard for one chain state x (DEVICE [P]):
 * one evaluation of the ray-lanes trace with per-task SM clock counters; each
 * warp's 32-ray task cost is split evenly over its rays (divergence included).
 * cost: HOST [R], caller's ray order, SM cycles.  Synchronous.  Requires the
 * ray-lanes mapping (a problem created with max_chains < 16); MT_EINVAL else. */
int mt_ray_cost(mt_problem *p, const float *x, float *cost);

/* Raw Philox4x32-10 words (device in ctr [n][4], out [n][4]; key host). */
int mt_philox(const uint32_t *ctr, uint32_t key0, uint32_t key1, uint32_t *out, int64_t n,
              mt_stream stream);
/* Same counters through cuRAND's curand_Philox4x32_10 (library cross-check). */
int mt_philox_curand(const uint32_t *ctr, uint32_t key0, uint32_t key1, uint32_t *out, int64_t n,
                     mt_stream stream);

/* ---- measurement ------------------------------------------------------- */

/* Start/stop recording CUDA events around every trace-kernel launch (on the
 * launching stream).  mt_timing_read returns the summed device time of the
 * trace launches (ms), their number, the chain x ray pairs they processed, and
 * the total number of kernels this problem launched since mt_timing_start. */
int mt_timing_start(mt_problem *p, int32_t max_records);
int mt_timing_read(mt_problem *p, double *trace_ms, int64_t *trace_launches, double *pairs,
                   int64_t *all_launches);

/* Trace work counters since mt_problem_create (synchronous; debugging and
 * bench reporting): `deferred` = chain x ray pairs the chain-lanes trace
 * kernel handed to its fp64 follow-up kernel (an ill-conditioned crossing,
 * SURVEY HP2, or more than 4 crossings of one surface); `defer_ms` = device
 * time of those follow-up launches while timing is on (mt_timing_start), also
 * included in mt_timing_read's trace_ms.  NULL outputs are skipped. */
int mt_trace_counters(mt_problem *p, int64_t *deferred, double *defer_ms);

/* FP32 FFMA throughput microbenchmark on `device` (TFLOP/s, FMA = 2 flops). */
int mt_measure_fp32_peak(int32_t device, double *tflops, double *sm_clock_mhz);

const char *mt_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* MT_H */
