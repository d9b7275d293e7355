// api.cu — C ABI of libmt (include/mt.h): problem validation and setup,
// per-evaluation orchestration (heights -> trace -> finish), leapfrog and
// HMC transitions, debug/parity exports, measurement hooks.
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <new>
#include <string>
#include <vector>

#include "mt_internal.cuh"

namespace {

thread_local std::string g_err;

int set_err(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_err(cudaError_t e, const char *where) {
  return set_err(MT_ECUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define CK(call)                                                  \
  do {                                                            \
    cudaError_t e_ = (call);                                      \
    if (e_ != cudaSuccess) return cuda_err(e_, #call);            \
  } while (0)

struct DevGuard {
  int prev = -1, want;
  explicit DevGuard(int d) : want(d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DevGuard() {
    if (prev >= 0 && prev != want) cudaSetDevice(prev);
  }
};

bool on_grid(double v) {  // multiple of 2^-12 with |v| < 2^11 (HP3)
  return fabs(v) < 2048.0 && floor(v * 4096.0) == v * 4096.0;
}

// Torus spectrum of Q = 4I - rA: σ² = mean(1/λ_ab),
// ln det Q = Σ ln λ_ab, λ_ab = 4 - 2r(cos 2πa/nx + cos 2πb/ny).
void torus(int nx, int ny, double r, double *sigma, double *logdet) {
  double s = 0, ld = 0;
  for (int a = 0; a < nx; a++)
    for (int b = 0; b < ny; b++) {
      double lam = 4.0 - 2.0 * r * (cos(2.0 * M_PI * a / nx) + cos(2.0 * M_PI * b / ny));
      s += 1.0 / lam;
      ld += log(lam);
    }
  *sigma = sqrt(s / ((double)nx * ny));
  *logdet = ld;
}

int check_ptr(const void *ptr, const char *name) {
  if (!ptr) return set_err(MT_EINVAL, "%s is NULL", name);
  return 0;
}

int check_chains(const mt_problem *p, int32_t C) {
  if (!p) return set_err(MT_EINVAL, "problem is NULL");
  if (C < 0) return set_err(MT_EINVAL, "C = %d < 0", C);
  if (C > p->max_chains) return set_err(MT_EINVAL, "C = %d > max_chains = %d", C, p->max_chains);
  return 0;
}

void free_all(mt_problem *p) {
  voxel_free(p);
  void *bufs[] = {p->d_X, p->d_Y, p->d_ray_a, p->d_ray_b, p->d_obase, p->d_perm, p->d_trav_off, p->d_trav, p->d_trav_geo, p->d_trav_km, p->d_rl_head, p->d_rl_code, p->d_rl_ovf, p->d_ovf_q, p->d_ovf_n, p->d_redo, p->d_H, p->d_Hlo, p->d_Hc, p->d_cl, p->d_cs, p->d_xw, p->d_minv, p->mb_red, p->mb_band, p->mb_ticket, p->d_xalt, p->d_fin_part, p->d_fin_ticket, p->d_G,
                  p->d_band, p->d_ll, p->d_x0, p->d_g0, p->d_mom, p->d_kin0, p->d_kin1, p->d_lp0};
  for (void *b : bufs)
    if (b) cudaFree(b);
  void *nb[] = {p->nuts_ws, p->nuts_lp, p->nuts_st, p->nuts_flags};
  for (void *b : nb)
    if (b) cudaFree(b);
  if (p->nuts_hflags) cudaFreeHost(p->nuts_hflags);
  for (auto e : p->ev_a) cudaEventDestroy(e);
  for (auto e : p->ev_b) cudaEventDestroy(e);
  for (auto e : p->ev_m) cudaEventDestroy(e);
}

}  // namespace

extern "C" {

const char *mt_last_error(void) { return g_err.c_str(); }

int mt_problem_create(const mt_problem_desc *d, mt_problem **out) {
  if (!out) return set_err(MT_EINVAL, "out is NULL");
  *out = nullptr;
  if (!d) return set_err(MT_EINVAL, "desc is NULL");
  // ---- validation (messages name the field) ----
  if (d->n_x < 3 || d->n_y < 3) return set_err(MT_EINVAL, "n_x, n_y must be >= 3 (torus stencil)");
  if (d->n_x > MT_MAX_AXIS || d->n_y > MT_MAX_AXIS || d->n_x * d->n_y > MT_MAX_NODES)
    return set_err(MT_EINVAL, "grid %dx%d exceeds %d nodes per surface", d->n_x, d->n_y, MT_MAX_NODES);
  if (check_ptr(d->node_x, "node_x") || check_ptr(d->node_y, "node_y")) return MT_EINVAL;
  for (int i = 0; i < d->n_x; i++) {
    if (!on_grid(d->node_x[i])) return set_err(MT_EINVAL, "node_x[%d] not on the 2^-12 m grid", i);
    if (i && !(d->node_x[i] > d->node_x[i - 1])) return set_err(MT_EINVAL, "node_x not increasing at %d", i);
  }
  for (int j = 0; j < d->n_y; j++) {
    if (!on_grid(d->node_y[j])) return set_err(MT_EINVAL, "node_y[%d] not on the 2^-12 m grid", j);
    if (j && !(d->node_y[j] > d->node_y[j - 1])) return set_err(MT_EINVAL, "node_y not increasing at %d", j);
  }
  if (!(d->z_top > 0) || !isfinite(d->z_top)) return set_err(MT_EINVAL, "z_top must be > 0");
  if (!(d->rho_muck >= 0 && d->rho_air >= 0 && d->rho_rock >= 0 && d->rho_ext >= 0))
    return set_err(MT_EINVAL, "densities must be >= 0");
  if (!(d->att_len > 0) || !isfinite(d->att_len)) return set_err(MT_EINVAL, "att_len must be > 0");
  for (int l = 0; l < 2; l++)
    if (!(d->car_r[l] >= 0.f && d->car_r[l] < 1.f)) return set_err(MT_EINVAL, "car_r[%d] not in [0,1)", l);
  if (d->n_det < 1 || check_ptr(d->det_xyz, "det_xyz")) return set_err(MT_EINVAL, "n_det < 1 or det_xyz NULL");
  float X0 = d->node_x[0], X1 = d->node_x[d->n_x - 1], Y0 = d->node_y[0], Y1 = d->node_y[d->n_y - 1];
  for (int k = 0; k < d->n_det; k++) {
    const float *o = d->det_xyz + 3 * k;
    if (!on_grid(o[0]) || !on_grid(o[1])) return set_err(MT_EINVAL, "det_xyz[%d] not on the 2^-12 m grid", k);
    if (!(o[0] > X0 && o[0] < X1 && o[1] > Y0 && o[1] < Y1))
      return set_err(MT_EINVAL, "detector %d not strictly inside the footprint", k);
    if (o[2] != 0.f) return set_err(MT_EINVAL, "detector %d: z must be 0 (the floor, R5)", k);
  }
  if (d->n_rays < 0) return set_err(MT_EINVAL, "n_rays < 0");
  if (d->n_rays > 0 && (check_ptr(d->ray_det, "ray_det") || check_ptr(d->ray_dir, "ray_dir") ||
                        check_ptr(d->ray_w, "ray_w") || check_ptr(d->counts, "counts")))
    return MT_EINVAL;
  if (d->ray_lo < 0 || d->ray_hi < d->ray_lo || d->ray_hi > d->n_rays)
    return set_err(MT_EINVAL, "ray shard [%lld, %lld) invalid", (long long)d->ray_lo, (long long)d->ray_hi);
  if (d->max_chains < 0) return set_err(MT_EINVAL, "max_chains < 0");
  if (d->noncentred && !d->sample_r) return set_err(MT_EINVAL, "noncentred requires sample_r");
  for (int64_t q = d->ray_lo; q < d->ray_hi; q++) {
    if (d->ray_det[q] < 0 || d->ray_det[q] >= d->n_det) return set_err(MT_EINVAL, "ray_det[%lld] out of range", (long long)q);
    const float *v = d->ray_dir + 3 * q;
    double nrm = sqrt((double)v[0] * v[0] + (double)v[1] * v[1] + (double)v[2] * v[2]);
    if (!(v[2] > 0.f)) return set_err(MT_EINVAL, "ray_dir[%lld]: d_z must be > 0", (long long)q);
    if (!(fabs(nrm - 1.0) <= 1e-6)) return set_err(MT_EINVAL, "ray_dir[%lld] not unit (|d| = %.9g)", (long long)q, nrm);
    if (!(d->ray_w[q] > 0.f) || !isfinite(d->ray_w[q])) return set_err(MT_EINVAL, "ray_w[%lld] must be > 0", (long long)q);
    if (d->counts[q] < 0 || d->counts[q] >= (1 << 24)) return set_err(MT_EINVAL, "counts[%lld] out of range", (long long)q);
  }
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (d->device < 0 || d->device >= ndev) return set_err(MT_EINVAL, "device %d not present (%d devices)", d->device, ndev);

  mt_problem *p = new (std::nothrow) mt_problem();
  if (!p) return set_err(MT_ENOMEM, "host allocation failed");
  DevGuard g(d->device);
  p->device = d->device;
  cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, d->device);
  p->sample_r = d->sample_r ? 1 : 0;
  p->ncp = d->noncentred ? 1 : 0;
  p->nx = d->n_x; p->ny = d->n_y; p->N = d->n_x * d->n_y; p->P = 2 * p->N + 2 * p->sample_r;
  p->R = d->ray_hi - d->ray_lo;
  p->ray_lo = d->ray_lo;
  p->max_chains = d->max_chains;
  p->z_top = d->z_top;
  p->car_r[0] = d->car_r[0]; p->car_r[1] = d->car_r[1];
  p->prior_on = d->ray_lo == 0;
  for (int l = 0; l < 2; l++) torus(p->nx, p->ny, d->car_r[l], &p->sigma[l], &p->logdetQ[l]);
  p->tc.nx = p->nx; p->tc.ny = p->ny; p->tc.N = p->N;
  p->tc.z_top = d->z_top;
  p->tc.k0 = d->rho_muck - d->rho_air;
  p->tc.k1 = d->rho_air - d->rho_rock;
  p->tc.inv_att = (float)(1.0 / (double)d->att_len);
  if (const char *e = getenv("MT_TRACE_K")) p->trace_k = atoi(e);
  if (const char *e = getenv("MT_TRACE_S")) p->trace_s = atoi(e);
  if (const char *e = getenv("MT_CHUNK")) p->chunk = atoi(e);
  if (const char *e = getenv("MT_CL_V")) p->cl_v = atoi(e);
  if (const char *e = getenv("MT_OVF_CAP")) p->ovf_cap = std::max(1, atoi(e));   // (tests: force the overflow path)

  // ---- per-ray constants in double (a0) ----
  std::vector<float4> ra(p->R), rb(p->R);
  std::vector<float> ob(p->R);
  double off = 0.0;
  const double Lam = d->att_len;
  for (int64_t q = 0; q < p->R; q++) {
    int64_t g_ = d->ray_lo + q;
    const float *o = d->det_xyz + 3 * d->ray_det[g_];
    const float *v = d->ray_dir + 3 * g_;
    double dx = v[0], dy = v[1], dz = v[2];
    double s_top = ((double)d->z_top - o[2]) / dz, s = s_top;
    if (dx > 0) s = fmin(s, ((double)X1 - o[0]) / dx);
    if (dx < 0) s = fmin(s, ((double)X0 - o[0]) / dx);
    if (dy > 0) s = fmin(s, ((double)Y1 - o[1]) / dy);
    if (dy < 0) s = fmin(s, ((double)Y0 - o[1]) / dy);
    double L_ext = s_top - s;
    double C = d->counts[g_], w = d->ray_w[g_];
    double obase = (double)d->rho_rock * s + (double)d->rho_ext * L_ext;
    double tb = log(w) - (C > 0 ? log(C) : 0.0) - obase / Lam;
    ra[q] = make_float4(o[0], o[1], v[0], v[1]);
    rb[q] = make_float4(v[2], (float)s, (float)tb, (float)C);
    ob[q] = (float)obase;
    off += (C > 0 ? C * log(C) : 0.0) - C - lgamma(C + 1.0);
  }
  p->loglik_offset = off;
  p->rho[0] = d->rho_muck; p->rho[1] = d->rho_air; p->rho[2] = d->rho_rock; p->rho[3] = d->rho_ext;
  p->att_len = d->att_len;
  p->hX.assign(d->node_x, d->node_x + p->nx);
  p->hY.assign(d->node_y, d->node_y + p->ny);

  // ---- internal ray order (performance only; results are order-independent
  // and per-ray outputs are mapped back): Morton order of the cell where the
  // ray reaches mid-height z_top/2, so rays processed together by a block
  // traverse the same band cells and their corner lines stay in L1.
  p->perm.resize(p->R);
  for (int64_t q = 0; q < p->R; q++) p->perm[q] = (int32_t)q;
  const char *ord = getenv("MT_RAY_ORDER");
  if (!(ord && atoi(ord) == 0)) {
    std::vector<uint64_t> key(p->R);
    // reference height of the order, as a fraction of z_top: mid-height for the chain
    // lanes (L2 locality of the band cells across a block's rays); lower for the ray
    // lanes, where lanes are rays and Morton neighbours there have more similar band
    // walks (configs[4]: 0.405 ms per trace at 0.5, 0.383 at 0.2-0.25, 0.415 at 0)
    double zf = p->max_chains >= 16 ? 0.5 : 0.22;
    if (const char *e = getenv("MT_ORDER_Z")) zf = atof(e);
    for (int64_t q = 0; q < p->R; q++) {
      double sm = fmin(zf * (double)d->z_top / rb[q].x, (double)rb[q].y);
      double px = ra[q].x + sm * ra[q].z, py = ra[q].y + sm * ra[q].w;
      int ci = (int)floor((px - X0) / ((double)X1 - X0) * (p->nx - 1));
      int cj = (int)floor((py - Y0) / ((double)Y1 - Y0) * (p->ny - 1));
      ci = ci < 0 ? 0 : (ci > p->nx - 2 ? p->nx - 2 : ci);
      cj = cj < 0 ? 0 : (cj > p->ny - 2 ? p->ny - 2 : cj);
      uint64_t m = 0;
      for (int b = 0; b < 16; b++) m |= (uint64_t)((ci >> b) & 1) << (2 * b) | (uint64_t)((cj >> b) & 1) << (2 * b + 1);
      key[q] = (m << 32) | (uint64_t)q;
    }
    // MT_ORDER_DET=1 (experiment): detector-major, the Morton order within each detector
    const char *od = getenv("MT_ORDER_DET");
    if (od && atoi(od) == 1) {
      const int32_t *det = d->ray_det + d->ray_lo;
      std::sort(p->perm.begin(), p->perm.end(), [&](int32_t a, int32_t b) {
        return det[a] != det[b] ? det[a] < det[b] : key[a] < key[b];
      });
    } else {
      std::sort(p->perm.begin(), p->perm.end(), [&](int32_t a, int32_t b) { return key[a] < key[b]; });
    }
    std::vector<float4> ra2(p->R), rb2(p->R);
    std::vector<float> ob2(p->R);
    for (int64_t k = 0; k < p->R; k++) {
      ra2[k] = ra[p->perm[k]]; rb2[k] = rb[p->perm[k]]; ob2[k] = ob[p->perm[k]];
    }
    ra.swap(ra2); rb.swap(rb2); ob.swap(ob2);
  }
  p->h_ra = ra;
  p->h_rb = rb;
  p->h_w.resize(p->R);
  for (int64_t k = 0; k < p->R; k++) p->h_w[k] = d->ray_w[d->ray_lo + p->perm[k]];
  p->inv_perm.resize(p->R);
  for (int64_t k = 0; k < p->R; k++) p->inv_perm[p->perm[k]] = (int32_t)k;

  // ---- device buffers ----
  size_t R = (size_t)(p->R > 0 ? p->R : 1), MC = (size_t)(p->max_chains > 0 ? p->max_chains : 1);
  size_t P = p->P;
  size_t MC32 = (MC + 31) / 32 * 32;   // chain-interleaved workspaces hold whole groups of 32
  cudaError_t e = cudaSuccess;
#define ALLOC(ptr, bytes)                                        \
  if (e == cudaSuccess) e = cudaMalloc((void **)&(ptr), (bytes));
  ALLOC(p->d_X, sizeof(float) * p->nx);
  ALLOC(p->d_Y, sizeof(float) * p->ny);
  ALLOC(p->d_ray_a, sizeof(float4) * R);
  ALLOC(p->d_ray_b, sizeof(float4) * R);
  ALLOC(p->d_obase, sizeof(float) * R);
  ALLOC(p->d_perm, sizeof(int32_t) * R);
  ALLOC(p->d_H, sizeof(float) * MC32 * P);
  ALLOC(p->d_Hlo, sizeof(float) * MC32 * P);
  // ray-lanes height copies: the ray lanes serve C < 16 unless MT_TRACE_K forces them
  const bool rl_any_c = p->trace_k != 0 && p->trace_k != 32;
  ALLOC(p->d_Hc, sizeof(float) * (rl_any_c || MC < 16 ? MC : 16) * P);
  ALLOC(p->d_cl, sizeof(float2) * (MC32 + 32) * 2 * p->N);   // (+32: whole 64-chain groups for k_cell_prep2)
  ALLOC(p->d_G, sizeof(macc) * MC32 * P);
  ALLOC(p->d_band, sizeof(float4) * MC);
  ALLOC(p->d_ll, sizeof(macc) * MC);
  ALLOC(p->d_x0, sizeof(float) * MC * P);
  ALLOC(p->d_g0, sizeof(float) * MC * P);
  ALLOC(p->d_mom, sizeof(float) * MC * P);
  ALLOC(p->d_kin0, sizeof(float) * MC);
  ALLOC(p->d_kin1, sizeof(float) * MC);
  ALLOC(p->d_lp0, sizeof(double) * MC);
  ALLOC(p->d_ovf_q, sizeof(float4) * (size_t)p->ovf_cap);
  ALLOC(p->d_ovf_n, sizeof(int) * 4);
  const size_t redo_words = (MC * R + 31) / 32;
  ALLOC(p->d_redo, sizeof(unsigned) * redo_words);
  ALLOC(p->d_cs, sizeof(double) * p->N);
  if (p->ncp) ALLOC(p->d_xw, sizeof(double) * MC * 2 * p->N);
  if (!getenv("MT_NO_FG")) {   // group-tiled K3: second x buffer, per-tile partials, tickets
    ALLOC(p->d_xalt, sizeof(float) * MC * P);
    ALLOC(p->d_fin_part, (size_t)48 * MC32 * ((p->N + 15) / 16));   // (tiles of >= 16 nodes)
    ALLOC(p->d_fin_ticket, sizeof(unsigned) * (MC32 / 32));
  }
  if (!getenv("MT_NO_MB")) {   // few-chain multi-block K3 / kick scratch (use_mb)
    ALLOC(p->mb_red, sizeof(double) * 16 * 3);
    ALLOC(p->mb_band, sizeof(unsigned) * 16 * 4);
    ALLOC(p->mb_ticket, sizeof(unsigned) * 16);
  }
#undef ALLOC
  if (e != cudaSuccess) {
    free_all(p);
    delete p;
    return e == cudaErrorMemoryAllocation ? set_err(MT_ENOMEM, "cudaMalloc: %s", cudaGetErrorString(e))
                                          : cuda_err(e, "cudaMalloc");
  }
  if (e == cudaSuccess) e = cudaMemcpy(p->d_X, d->node_x, sizeof(float) * p->nx, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(p->d_Y, d->node_y, sizeof(float) * p->ny, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && p->R > 0) e = cudaMemcpy(p->d_ray_a, ra.data(), sizeof(float4) * p->R, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && p->R > 0) e = cudaMemcpy(p->d_ray_b, rb.data(), sizeof(float4) * p->R, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && p->R > 0) e = cudaMemcpy(p->d_obase, ob.data(), sizeof(float) * p->R, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && p->R > 0) e = cudaMemcpy(p->d_perm, p->perm.data(), sizeof(int32_t) * p->R, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(p->d_G, 0, sizeof(macc) * MC32 * P);
  if (e == cudaSuccess) e = cudaMemset(p->d_H, 0, sizeof(float) * MC32 * P);
  if (e == cudaSuccess) e = cudaMemset(p->d_Hlo, 0, sizeof(float) * MC32 * P);
  if (e == cudaSuccess) e = cudaMemset(p->d_ll, 0, sizeof(macc) * MC);
  if (e == cudaSuccess && p->d_fin_ticket) e = cudaMemset(p->d_fin_ticket, 0, sizeof(unsigned) * (MC32 / 32));
  if (e == cudaSuccess) e = cudaMemset(p->d_ovf_n, 0, sizeof(int) * 4);
  if (e == cudaSuccess) e = cudaMemset(p->d_redo, 0, sizeof(unsigned) * redo_words);
  if (e == cudaSuccess && p->mb_red) {
    std::vector<unsigned> b(64);
    for (int k = 0; k < 16; k++) { b[4 * k] = b[4 * k + 2] = 0x7f7fffffu; b[4 * k + 1] = b[4 * k + 3] = 0u; }
    e = cudaMemset(p->mb_red, 0, sizeof(double) * 48);
    if (e == cudaSuccess) e = cudaMemset(p->mb_ticket, 0, sizeof(unsigned) * 16);
    if (e == cudaSuccess) e = cudaMemcpy(p->mb_band, b.data(), sizeof(unsigned) * 64, cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess) {   // torus spectrum table c_ab = 2(cos 2πa/n_x + cos 2πb/n_y) (sample_r)
    std::vector<double> cs(p->N);
    for (int a = 0; a < p->nx; a++)
      for (int b = 0; b < p->ny; b++)
        cs[a * p->ny + b] = 2.0 * (cos(2.0 * M_PI * a / p->nx) + cos(2.0 * M_PI * b / p->ny));
    e = cudaMemcpy(p->d_cs, cs.data(), sizeof(double) * p->N, cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = build_traversal(p);   // a2, once per problem (exact predicates)
  if (e != cudaSuccess) {
    free_all(p);
    delete p;
    return cuda_err(e, "mt_problem_create upload/traversal");
  }
  *out = p;
  return MT_OK;
}

int mt_problem_destroy(mt_problem *p) {
  if (!p) return MT_OK;
  DevGuard g(p->device);
  cudaDeviceSynchronize();
  comm_detach(p);
  free_all(p);
  delete p;
  return MT_OK;
}

int32_t mt_num_params(const mt_problem *p) { return p ? p->P : 0; }
int64_t mt_num_rays(const mt_problem *p) { return p ? p->R : 0; }
double mt_loglik_offset(const mt_problem *p) { return p ? p->loglik_offset : 0.0; }

int mt_prior_constants(const mt_problem *p, double sigma[2], double logdetQ[2]) {
  if (!p || !sigma || !logdetQ) return set_err(MT_EINVAL, "NULL argument");
  for (int l = 0; l < 2; l++) { sigma[l] = p->sigma[l]; logdetQ[l] = p->logdetQ[l]; }
  return MT_OK;
}

// Ray sharding with an attached communicator: one evaluation = trace of this
// shard + chain rule / prior (shard 0) -> partial [logp, grad] -> in-stream
// NCCL SUM all-reduce -> full [logp, grad] on every rank.
static int eval_sharded(mt_problem *p, int C, float *x, double *logp, float *grad, int32_t *status,
                        cudaStream_t s) {
  CK(launch_trace(p, TRACE_LL, C, p->d_H, p->d_band, p->d_G, p->d_ll, nullptr, nullptr, s));
  CK(launch_finish(p, FIN_PLAIN, C, x, grad, logp, status, nullptr, nullptr, nullptr, s));
  if (!p->comm) return MT_OK;   // (the non-centred mode uses this unfused path on one shard too)
  std::string why;
  if (comm_allreduce_logp_grad(p, C, logp, grad, s, why) != cudaSuccess)
    return set_err(MT_ENCCL, "ncclAllReduce: %s", why.c_str());
  return MT_OK;
}

int mt_logpost_grad(mt_problem *p, int32_t C, const float *x, double *logp, float *grad,
                    int32_t *status, mt_stream stream) {
  if (int r = check_chains(p, C)) return r;
  if (C == 0) return MT_OK;
  if (check_ptr(x, "x") || check_ptr(logp, "logp") || check_ptr(grad, "grad")) return MT_EINVAL;
  DevGuard g(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  CK(launch_heights(p, C, x, p->d_H, p->d_band, s));
  if (p->comm || p->ncp || use_mb(p, C)) return eval_sharded(p, C, const_cast<float *>(x), logp, grad, status, s);
  CK(launch_trace(p, TRACE_LL, C, p->d_H, p->d_band, p->d_G, p->d_ll, nullptr, nullptr, s));
  CK(launch_finish(p, FIN_PLAIN, C, const_cast<float *>(x), grad, logp, status, nullptr, nullptr,
                   nullptr, s));
  return MT_OK;
}

// L leapfrog evaluations with all-reduced gradients (x, mom already carry the
// first half kick + drift and d_H the heights of the drifted x).
static int leapfrog_sharded(mt_problem *p, int C, float *x, float *mom, double *logp, float *grad,
                            int32_t *status, const float *eps, int L, cudaStream_t s) {
  for (int step = 1; step <= L; step++) {
    if (int r = eval_sharded(p, C, x, logp, grad, status, s)) return r;
    if (step < L) CK(launch_kick(p, KICK_FULL_DRIFT, C, x, mom, grad, eps, nullptr, s));
    else CK(launch_kick(p, KICK_HALF_LAST, C, x, mom, grad, eps, p->d_kin1, s));
  }
  return MT_OK;
}

// L fused evaluations + kicks (x, mom already carry the first half kick + drift).
// The group-tiled K3 reads x from one buffer and writes the drifted x to the
// other (the caller's block and d_xalt alternate), so no tile reads a halo node
// another tile has already updated; the last step (no drift) leaves x in the
// caller's block.
static int leapfrog_fused(mt_problem *p, int C, float *x, float *mom, double *logp, float *grad,
                          int32_t *status, const float *eps, int L, cudaStream_t s) {
  const bool pp = use_fg(p, C);
  float *cur = x;
  for (int step = 1; step <= L; step++) {
    CK(launch_trace(p, TRACE_LL, C, p->d_H, p->d_band, p->d_G, p->d_ll, nullptr, nullptr, s));
    float *dst = step < L && pp ? (cur == x ? p->d_xalt : x) : x;
    CK(launch_finish(p, step < L ? FIN_STEP : FIN_LAST, C, dst, grad, logp, status, mom, eps, p->d_kin1, s, cur));
    if (step < L) cur = dst;
  }
  return MT_OK;
}

int mt_leapfrog(mt_problem *p, int32_t C, float *x, float *mom, double *logp, float *grad,
                const float *eps, int32_t L, mt_stream stream) {
  if (int r = check_chains(p, C)) return r;
  if (L < 0) return set_err(MT_EINVAL, "L = %d < 0", L);
  if (C == 0 || L == 0) return MT_OK;
  if (check_ptr(x, "x") || check_ptr(mom, "p") || check_ptr(logp, "logp") || check_ptr(grad, "grad") ||
      check_ptr(eps, "eps"))
    return MT_EINVAL;
  DevGuard g(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  CK(launch_kick_drift(p, C, x, mom, grad, eps, s));
  if (p->comm || p->ncp || use_mb(p, C)) return leapfrog_sharded(p, C, x, mom, logp, grad, nullptr, eps, L, s);
  if (int r = leapfrog_fused(p, C, x, mom, logp, grad, nullptr, eps, L, s)) return r;
  return MT_OK;
}

int mt_draw_momenta(mt_problem *p, int32_t C, float *mom, uint64_t seed, uint64_t iter,
                    uint64_t chain_offset, mt_stream stream) {
  if (int r = check_chains(p, C)) return r;
  if (C == 0) return MT_OK;
  if (check_ptr(mom, "p")) return MT_EINVAL;
  DevGuard g(p->device);
  CK(launch_momenta(p, C, mom, seed, iter, chain_offset, (cudaStream_t)stream));
  return MT_OK;
}

int mt_hmc_step(mt_problem *p, int32_t C, float *x, double *logp, float *grad, const float *eps,
                int32_t L, uint64_t seed, uint64_t iter, uint64_t chain_offset, float *accept_prob,
                int32_t *accepted, int32_t *status, mt_stream stream) {
  if (int r = check_chains(p, C)) return r;
  if (L < 1) return set_err(MT_EINVAL, "L = %d < 1", L);
  if (C == 0) return MT_OK;
  if (check_ptr(x, "x") || check_ptr(logp, "logp") || check_ptr(grad, "grad") || check_ptr(eps, "eps") ||
      check_ptr(accept_prob, "accept_prob") || check_ptr(accepted, "accepted"))
    return MT_EINVAL;
  DevGuard g(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  CK(launch_hmc_begin(p, C, x, logp, grad, eps, seed, iter, chain_offset, s));
  if (p->comm || p->ncp || use_mb(p, C)) {
    if (int r = leapfrog_sharded(p, C, x, p->d_mom, logp, grad, status, eps, L, s)) return r;
    CK(launch_hmc_end(p, C, x, logp, grad, seed, iter, chain_offset, accept_prob, accepted, status, s));
    return MT_OK;
  }
  if (int r = leapfrog_fused(p, C, x, p->d_mom, logp, grad, status, eps, L, s)) return r;
  CK(launch_hmc_end(p, C, x, logp, grad, seed, iter, chain_offset, accept_prob, accepted, status, s));
  return MT_OK;
}

int mt_nuts_record(mt_problem *p, float *th, float *g, double *lp, int32_t max_leaves) {
  if (!p) return set_err(MT_EINVAL, "problem is NULL");
  if (th && (!g || !lp || max_leaves < 0)) return set_err(MT_EINVAL, "bad record buffers");
  p->nuts_rec_th = th;
  p->nuts_rec_g = th ? g : nullptr;
  p->nuts_rec_lp = th ? lp : nullptr;
  p->nuts_rec_max = th ? max_leaves : 0;
  return MT_OK;
}

int mt_nuts_step(mt_problem *p, int32_t C, float *x, double *logp, float *grad, const float *eps,
                 int32_t max_depth, uint64_t seed, uint64_t iter, uint64_t chain_offset, float *accept_stat,
                 int32_t *depth, int32_t *n_leaves, int32_t *status, mt_stream stream) {
  if (int r = check_chains(p, C)) return r;
  if (p->ncp) return set_err(MT_EINVAL, "mt_nuts_step: not available with noncentred");
  if (max_depth < 1 || max_depth > MT_NUTS_MAX_DEPTH)
    return set_err(MT_EINVAL, "max_depth = %d not in [1, %d]", max_depth, MT_NUTS_MAX_DEPTH);
  if (C == 0) return MT_OK;
  if (check_ptr(x, "x") || check_ptr(logp, "logp") || check_ptr(grad, "grad") || check_ptr(eps, "eps") ||
      check_ptr(accept_stat, "accept_stat"))
    return MT_EINVAL;
  DevGuard g(p->device);
  std::string why;
  cudaError_t e = run_nuts(p, C, x, logp, grad, eps, max_depth, seed, iter, chain_offset, accept_stat, depth,
                           n_leaves, status, (cudaStream_t)stream, why);
  if (!why.empty()) return set_err(MT_ENCCL, "ncclAllReduce: %s", why.c_str());
  if (e == cudaErrorMemoryAllocation) return set_err(MT_ENOMEM, "NUTS workspace: %s", cudaGetErrorString(e));
  CK(e);
  return MT_OK;
}

int mt_comm_unique_id(void *uid128) {
  if (!uid128) return set_err(MT_EINVAL, "uid buffer is NULL");
  std::string why;
  if (!comm_unique_id(uid128, why)) return set_err(MT_ENCCL, "ncclGetUniqueId: %s", why.c_str());
  return MT_OK;
}

int mt_attach_comm(mt_problem *p, const void *uid128, int32_t rank, int32_t world) {
  if (!p || !uid128) return set_err(MT_EINVAL, "NULL argument");
  if (world < 1 || rank < 0 || rank >= world) return set_err(MT_EINVAL, "rank %d / world %d", rank, world);
  DevGuard g(p->device);
  std::string why;
  if (!comm_attach(p, uid128, rank, world, why)) return set_err(MT_ENCCL, "ncclCommInitRank: %s", why.c_str());
  return MT_OK;
}

int mt_detach_comm(mt_problem *p) {
  if (!p) return set_err(MT_EINVAL, "problem is NULL");
  DevGuard g(p->device);
  cudaDeviceSynchronize();
  comm_detach(p);
  return MT_OK;
}

int mt_stats_update(mt_problem *p, int32_t C, const float *x, const float *accept_prob,
                    int32_t n_prev, float *mean, float *m2, uint64_t *acc_fixed, mt_stream stream) {
  if (int r = check_chains(p, C)) return r;
  if (n_prev < 0) return set_err(MT_EINVAL, "n_prev < 0");
  if ((x || mean || m2) && !(x && mean && m2)) return set_err(MT_EINVAL, "x, mean, m2 must all be given");
  if ((accept_prob != nullptr) != (acc_fixed != nullptr))
    return set_err(MT_EINVAL, "accept_prob and acc_fixed must both be given");
  DevGuard g(p->device);
  CK(launch_stats(p, C, x, accept_prob, n_prev, mean, m2,
                  reinterpret_cast<unsigned long long *>(acc_fixed), (cudaStream_t)stream));
  return MT_OK;
}

int mt_rhat_partials(mt_problem *p, int32_t C, const float *mean, const float *m2, int32_t n,
                     double *out, mt_stream stream) {
  if (int r = check_chains(p, C)) return r;
  if (check_ptr(mean, "mean") || check_ptr(m2, "m2") || check_ptr(out, "out")) return MT_EINVAL;
  if (n < 2) return set_err(MT_EINVAL, "n = %d < 2", n);
  DevGuard g(p->device);
  CK(launch_rhat_partials(p, C, mean, m2, n, out, (cudaStream_t)stream));
  return MT_OK;
}

int mt_nested_rhat_partials(mt_problem *p, int32_t C, int32_t M, const float *mean, const float *m2, int32_t n,
                            double *out, mt_stream stream) {
  if (int r = check_chains(p, C)) return r;
  if (check_ptr(mean, "mean") || check_ptr(m2, "m2") || check_ptr(out, "out")) return MT_EINVAL;
  if (M < 1 || C % M) return set_err(MT_EINVAL, "C = %d not a multiple of the super-chain size M = %d", C, M);
  if (n < 1) return set_err(MT_EINVAL, "n = %d < 1", n);
  DevGuard g(p->device);
  CK(launch_nested_rhat_partials(p, C, M, mean, m2, n, out, (cudaStream_t)stream));
  return MT_OK;
}

int mt_summary_update(mt_problem *p, int32_t C, const float *x, const double *logp, int32_t nz, float gap,
                      double *acc, float *map_x, double *map_logp, mt_stream stream) {
  if (int r = check_chains(p, C)) return r;
  if (C == 0) return MT_OK;
  if (nz < 1) return set_err(MT_EINVAL, "nz = %d < 1", nz);
  if (check_ptr(x, "x") || check_ptr(acc, "acc")) return MT_EINVAL;
  if ((map_x != nullptr) != (map_logp != nullptr) || (map_x && !logp))
    return set_err(MT_EINVAL, "map_x, map_logp and logp go together");
  DevGuard g(p->device);
  CK(launch_summary(p, C, x, logp, nz, gap, acc, map_x, map_logp, (cudaStream_t)stream));
  return MT_OK;
}

int mt_set_step_counters(mt_problem *p, uint64_t *iter, int32_t *n_prev) {
  if (!p) return set_err(MT_EINVAL, "problem is NULL");
  p->d_iter = iter;
  p->d_nprev = n_prev;
  return MT_OK;
}

int mt_summary_finalize(mt_problem *p, int32_t nz, const double *acc, double *out, mt_stream stream) {
  if (!p) return set_err(MT_EINVAL, "problem is NULL");
  if (nz < 1) return set_err(MT_EINVAL, "nz = %d < 1", nz);
  if (check_ptr(acc, "acc") || check_ptr(out, "out")) return MT_EINVAL;
  DevGuard g(p->device);
  CK(launch_summary_finalize(p, nz, acc, out, (cudaStream_t)stream));
  return MT_OK;
}

int mt_heights(mt_problem *p, int32_t C, const float *x, float *H, mt_stream stream) {
  if (int r = check_chains(p, C)) return r;
  if (C == 0) return MT_OK;
  if (check_ptr(x, "x") || check_ptr(H, "H")) return MT_EINVAL;
  DevGuard g(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  CK(launch_heights(p, C, x, p->d_H, p->d_band, s));
  CK(launch_tile(p, C, p->d_H, H, 0, s));
  return MT_OK;
}

// band of caller-given heights (min/max per surface) through the K3 reduce
// path is not needed: compute it with a tiny kernel-free approach by reusing
// the heights kernel's band reduction on H directly.
__global__ void k_band_of(const float *H, int N, float4 *band) {
  const float *Hc = H + (size_t)blockIdx.x * 2 * N;
  float a = 3e38f, b = -3e38f, c = 3e38f, d = -3e38f;
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    a = fminf(a, Hc[k]); b = fmaxf(b, Hc[k]);
    c = fminf(c, Hc[N + k]); d = fmaxf(d, Hc[N + k]);
  }
  __shared__ float sh[4][256];
  sh[0][threadIdx.x] = a; sh[1][threadIdx.x] = b; sh[2][threadIdx.x] = c; sh[3][threadIdx.x] = d;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)blockDim.x; k++) {
      a = fminf(a, sh[0][k]); b = fmaxf(b, sh[1][k]); c = fminf(c, sh[2][k]); d = fmaxf(d, sh[3][k]);
    }
    band[blockIdx.x] = make_float4(a, b, c, d);
  }
}

int mt_loglik_heights(mt_problem *p, int32_t C, const float *H, double *ll, float *dldH,
                      mt_stream stream) {
  if (int r = check_chains(p, C)) return r;
  if (C == 0) return MT_OK;
  if (check_ptr(H, "H") || check_ptr(ll, "ll") || check_ptr(dldH, "dldH")) return MT_EINVAL;
  DevGuard g(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  k_band_of<<<C, 256, 0, s>>>(H, p->N, p->d_band);
  p->all_launches++;
  CK(cudaGetLastError());
  CK(launch_tile(p, C, H, p->d_H, 1, s));
  CK(cudaMemsetAsync(p->d_Hlo, 0, sizeof(float) * ((size_t)(C + 31) / 32 * 32) * p->P, s));   // exact fp32 heights
  CK(launch_trace(p, TRACE_LL, C, p->d_H, p->d_band, p->d_G, p->d_ll, nullptr, nullptr, s));
  CK(launch_take_acc(p, C, dldH, ll, s));
  return MT_OK;
}

int mt_path_lengths(mt_problem *p, int32_t C, const float *H, float *L, float *O, mt_stream stream) {
  if (int r = check_chains(p, C)) return r;
  if (C == 0) return MT_OK;
  if (check_ptr(H, "H") || check_ptr(L, "L") || check_ptr(O, "O")) return MT_EINVAL;
  DevGuard g(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  k_band_of<<<C, 256, 0, s>>>(H, p->N, p->d_band);
  p->all_launches++;
  CK(cudaGetLastError());
  CK(launch_tile(p, C, H, p->d_H, 1, s));
  CK(cudaMemsetAsync(p->d_Hlo, 0, sizeof(float) * ((size_t)(C + 31) / 32 * 32) * p->P, s));   // exact fp32 heights
  CK(launch_trace(p, TRACE_PATH, C, p->d_H, p->d_band, nullptr, nullptr, L, O, s));
  return MT_OK;
}

int mt_ray_work(mt_problem *p, const float *x, int32_t *work) {
  if (!p || !work) return set_err(MT_EINVAL, "NULL problem or work");
  if (check_ptr(x, "x")) return MT_EINVAL;
  if (p->max_chains < 1) return set_err(MT_EINVAL, "max_chains < 1");
  DevGuard g(p->device);
  CK(cudaDeviceSynchronize());
  CK(launch_heights(p, 1, x, p->d_H, p->d_band, 0));
  float4 bd;
  CK(cudaMemcpy(&bd, p->d_band, sizeof(float4), cudaMemcpyDeviceToHost));
  std::vector<int32_t> io(p->R + 1);
  std::vector<int2> cells(p->trav_cells > 0 ? p->trav_cells : 1);
  if (p->R > 0) CK(cudaMemcpy(io.data(), p->d_trav_off, sizeof(int32_t) * (p->R + 1), cudaMemcpyDeviceToHost));
  if (p->trav_cells > 0) CK(cudaMemcpy(cells.data(), p->d_trav, sizeof(int2) * p->trav_cells, cudaMemcpyDeviceToHost));
  for (int64_t k = 0; k < p->R; k++) {   // internal ray k
    const float dz = p->h_rb[k].x;
    int32_t n = 0;
    float s = 0.f;
    for (int32_t m = io[k]; m < io[k + 1]; m++) {
      float so;
      memcpy(&so, &cells[m].y, sizeof so);
      if (so * dz > bd.x && s * dz < bd.w) n++;
      s = so;
    }
    work[p->perm[k]] = n;
  }
  return MT_OK;
}

int mt_ray_cost(mt_problem *p, const float *x, float *cost) {
  if (!p || !cost) return set_err(MT_EINVAL, "NULL problem or cost");
  if (check_ptr(x, "x")) return MT_EINVAL;
  if (p->max_chains >= 16 || p->trace_k == 32 || p->vx.nz > 0)
    return set_err(MT_EINVAL, "mt_ray_cost needs the ray-lanes trace (max_chains < 16, exact model)");
  DevGuard g(p->device);
  CK(cudaDeviceSynchronize());
  const int64_t ntask = (p->R + 31) / 32 + 1;
  unsigned long long *d_cost = nullptr;
  CK(cudaMalloc(&d_cost, sizeof(unsigned long long) * ntask));
  cudaError_t e = cudaMemset(d_cost, 0, sizeof(unsigned long long) * ntask);
  if (e == cudaSuccess) e = launch_heights(p, 1, x, p->d_H, p->d_band, 0);
  if (e == cudaSuccess) e = launch_trace(p, TRACE_LL, 1, p->d_H, p->d_band, p->d_G, p->d_ll, nullptr, nullptr, 0, d_cost);
  if (e == cudaSuccess) e = cudaMemsetAsync(p->d_G, 0, sizeof(macc) * 32 * (size_t)p->P, 0);
  if (e == cudaSuccess) e = cudaMemsetAsync(p->d_ll, 0, sizeof(macc), 0);
  std::vector<unsigned long long> h(ntask);
  if (e == cudaSuccess) e = cudaMemcpy(h.data(), d_cost, sizeof(unsigned long long) * ntask, cudaMemcpyDeviceToHost);
  cudaFree(d_cost);
  if (e != cudaSuccess) return cuda_err(e, "mt_ray_cost");
  for (int64_t k = 0; k < p->R; k++) cost[p->perm[k]] = (float)h[k >> 5] / 32.f;   // internal ray k
  return MT_OK;
}

int mt_traversal_all(mt_problem *p, int64_t *off, int32_t *ij, float *s_out) {
  if (!p || !off) return set_err(MT_EINVAL, "NULL problem or off");
  if (ij && !s_out) return set_err(MT_EINVAL, "s_out is NULL");
  DevGuard g(p->device);
  CK(cudaDeviceSynchronize());
  std::vector<int32_t> io(p->R + 1);
  if (p->R > 0) CK(cudaMemcpy(io.data(), p->d_trav_off, sizeof(int32_t) * (p->R + 1), cudaMemcpyDeviceToHost));
  off[0] = 0;
  for (int64_t q = 0; q < p->R; q++) {   // caller ray q = internal ray inv_perm[q]
    const int64_t k = p->inv_perm[q];
    off[q + 1] = off[q] + (io[k + 1] - io[k]);
  }
  if (!ij || p->R == 0) return MT_OK;
  std::vector<int2> cells(p->trav_cells > 0 ? p->trav_cells : 1);
  if (p->trav_cells > 0) CK(cudaMemcpy(cells.data(), p->d_trav, sizeof(int2) * p->trav_cells, cudaMemcpyDeviceToHost));
  for (int64_t q = 0; q < p->R; q++) {
    const int64_t k = p->inv_perm[q];
    int64_t o = off[q];
    for (int32_t m = io[k]; m < io[k + 1]; m++, o++) {
      ij[2 * o] = cell_i(cells[m].x);
      ij[2 * o + 1] = cell_j(cells[m].x);
      memcpy(&s_out[o], &cells[m].y, sizeof(float));
    }
  }
  return MT_OK;
}

int mt_debug_traversal(mt_problem *p, int64_t ray, int32_t *ij, float *s_in, float *s_out,
                       int32_t cap, int32_t *n) {
  if (!p) return set_err(MT_EINVAL, "problem is NULL");
  if (ray < 0 || ray >= p->R) return set_err(MT_EINVAL, "ray %lld out of range", (long long)ray);
  if (cap < 0 || !n || (cap > 0 && (!ij || !s_in || !s_out))) return set_err(MT_EINVAL, "bad output buffers");
  DevGuard g(p->device);
  // the stored traversal the trace kernels read (built by the exact device DDA)
  int32_t off[2];
  CK(cudaMemcpy(off, p->d_trav_off + p->inv_perm[ray], sizeof(int32_t) * 2, cudaMemcpyDeviceToHost));
  *n = (int32_t)(off[1] - off[0]);
  int m = *n < cap ? *n : cap;
  if (m > 0) {
    std::vector<int2> cells(m);
    CK(cudaMemcpy(cells.data(), p->d_trav + off[0], sizeof(int2) * m, cudaMemcpyDeviceToHost));
    float prev = 0.f;
    for (int k = 0; k < m; k++) {
      ij[2 * k] = cell_i(cells[k].x);
      ij[2 * k + 1] = cell_j(cells[k].x);
      float so;
      memcpy(&so, &cells[k].y, sizeof so);
      s_in[k] = prev;
      s_out[k] = so;
      prev = so;
    }
  }
  return MT_OK;
}

int mt_philox(const uint32_t *ctr, uint32_t key0, uint32_t key1, uint32_t *out, int64_t n,
              mt_stream stream) {
  if (n < 0 || (n > 0 && (!ctr || !out))) return set_err(MT_EINVAL, "bad philox arguments");
  CK(launch_philox(ctr, key0, key1, out, n, 0, (cudaStream_t)stream));
  return MT_OK;
}

int mt_philox_curand(const uint32_t *ctr, uint32_t key0, uint32_t key1, uint32_t *out, int64_t n,
                     mt_stream stream) {
  if (n < 0 || (n > 0 && (!ctr || !out))) return set_err(MT_EINVAL, "bad philox arguments");
  CK(launch_philox(ctr, key0, key1, out, n, 1, (cudaStream_t)stream));
  return MT_OK;
}

int mt_timing_start(mt_problem *p, int32_t max_records) {
  if (!p || max_records < 0) return set_err(MT_EINVAL, "bad timing arguments");
  DevGuard g(p->device);
  while ((int)p->ev_a.size() < max_records) {
    cudaEvent_t a, b, m;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventCreate(&m));
    p->ev_a.push_back(a);
    p->ev_b.push_back(b);
    p->ev_m.push_back(m);
  }
  p->n_rec = 0;
  p->trace_launches = 0;
  p->all_launches = 0;
  p->pairs = 0;
  p->timing = true;
  return MT_OK;
}

int mt_timing_read(mt_problem *p, double *trace_ms, int64_t *trace_launches, double *pairs,
                   int64_t *all_launches) {
  if (!p) return set_err(MT_EINVAL, "problem is NULL");
  DevGuard g(p->device);
  double tot = 0, def = 0;
  for (int k = 0; k < p->n_rec; k++) {
    CK(cudaEventSynchronize(p->ev_b[k]));
    float ms = 0, md = 0;
    CK(cudaEventElapsedTime(&ms, p->ev_a[k], p->ev_b[k]));
    CK(cudaEventElapsedTime(&md, p->ev_m[k], p->ev_b[k]));
    tot += ms;
    def += md;
  }
  p->defer_ms = def;
  if (trace_ms) *trace_ms = tot;
  if (trace_launches) *trace_launches = p->trace_launches;
  if (pairs) *pairs = p->pairs;
  if (all_launches) *all_launches = p->all_launches;
  p->timing = false;
  return MT_OK;
}

int mt_trace_counters(mt_problem *p, int64_t *deferred, double *defer_ms) {
  if (!p) return set_err(MT_EINVAL, "problem is NULL");
  DevGuard g(p->device);
  if (deferred) {
    unsigned long long v = 0;
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(&v, p->d_ovf_n + 2, sizeof v, cudaMemcpyDeviceToHost));
    *deferred = (int64_t)v;
  }
  if (defer_ms) *defer_ms = p->defer_ms;
  return MT_OK;
}

int mt_set_inverse_mass(mt_problem *p, const float *minv, int32_t n) {
  if (!p) return set_err(MT_EINVAL, "problem is NULL");
  DevGuard g(p->device);
  if (!minv) {   // back to the identity mass
    CK(cudaDeviceSynchronize());
    if (p->d_minv) cudaFree(p->d_minv);
    p->d_minv = nullptr;
    return MT_OK;
  }
  if (n != p->P) return set_err(MT_EINVAL, "n = %d != P = %d", n, p->P);
  // synchronous on the whole device (mt.h): the producer of minv may run on any stream, and
  // kernels already queued may still read the old d_minv
  CK(cudaDeviceSynchronize());
  std::vector<float> h(p->P);
  CK(cudaMemcpy(h.data(), minv, sizeof(float) * p->P, cudaMemcpyDeviceToHost));
  for (int k = 0; k < p->P; k++)
    if (!(h[k] > 0.f) || !isfinite(h[k])) return set_err(MT_EINVAL, "minv[%d] = %g must be finite and > 0", k, h[k]);
  if (!p->d_minv) {
    cudaError_t e = cudaMalloc((void **)&p->d_minv, sizeof(float) * p->P);
    if (e != cudaSuccess) return set_err(MT_ENOMEM, "cudaMalloc: %s", cudaGetErrorString(e));
  }
  CK(cudaMemcpy(p->d_minv, h.data(), sizeof(float) * p->P, cudaMemcpyHostToDevice));
  return MT_OK;
}

int mt_voxel_model(mt_problem *p, int32_t n_z, float gamma, float tau, const float *H_ref) {
  if (!p) return set_err(MT_EINVAL, "problem is NULL");
  if (n_z < 0 || n_z > 4096) return set_err(MT_EINVAL, "n_z = %d not in [0, 4096]", n_z);
  if (n_z > 0) {
    if (!(gamma > 0.f) || !isfinite(gamma)) return set_err(MT_EINVAL, "gamma must be > 0");
    if (!(tau >= 0.f && tau < 1.f)) return set_err(MT_EINVAL, "tau not in [0, 1)");
    if (check_ptr(H_ref, "H_ref")) return MT_EINVAL;
    for (int k = 0; k < 2 * p->N; k++)
      if (!isfinite(H_ref[k])) return set_err(MT_EINVAL, "H_ref[%d] not finite", k);
    if ((int64_t)p->N * n_z > ((int64_t)1 << 23) || p->R > ((int64_t)1 << 23))
      return set_err(MT_EINVAL, "voxel model: at most 2^23 voxels and 2^23 rays per shard");
  }
  DevGuard g(p->device);
  CK(cudaDeviceSynchronize());
  cudaError_t e = voxel_setup(p, n_z, gamma, tau, H_ref);
  if (e == cudaErrorMemoryAllocation) return set_err(MT_ENOMEM, "voxel model: cudaMalloc failed");
  if (e != cudaSuccess) return cuda_err(e, "voxel_setup");
  return MT_OK;
}

int mt_voxel_info(const mt_problem *p, int32_t *n_z, int64_t *nnz, int64_t *n_grid) {
  if (!p) return set_err(MT_EINVAL, "problem is NULL");
  if (n_z) *n_z = p->vx.nz;
  if (nnz) *nnz = p->vx.nnz;
  if (n_grid) *n_grid = p->vx.ng;
  return MT_OK;
}

int mt_voxel_counters(mt_problem *p, uint64_t *gathered_bytes) {
  if (!p || !gathered_bytes) return set_err(MT_EINVAL, "NULL argument");
  *gathered_bytes = 0;
  if (!p->vx.gathered) return MT_OK;
  DevGuard g(p->device);
  CK(cudaDeviceSynchronize());
  unsigned long long v = 0;
  CK(cudaMemcpy(&v, p->vx.gathered, sizeof v, cudaMemcpyDeviceToHost));
  *gathered_bytes = v;
  return MT_OK;
}

int mt_measure_l2_gather(int32_t device, int64_t bytes, double *gbs) {
  if (!gbs || bytes < (1 << 20)) return set_err(MT_EINVAL, "gbs NULL or bytes < 1 MiB");
  DevGuard g(device);
  CK(run_l2_gather_peak(device, (size_t)bytes, gbs));
  return MT_OK;
}

int mt_measure_fp32_peak(int32_t device, double *tflops, double *sm_clock_mhz) {
  if (!tflops || !sm_clock_mhz) return set_err(MT_EINVAL, "NULL argument");
  DevGuard g(device);
  CK(run_fp32_peak(device, tflops, sm_clock_mhz));
  return MT_OK;
}

}  // extern "C"
