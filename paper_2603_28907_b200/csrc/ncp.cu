// ncp.cu — the non-centred CAR parameterisation x = Q(r)^{-1/2} z (SURVEY
// §8(f) f2, reading R13d): per-chain 2-D FFT / DFT circulant
// applications in fp64 shared memory, on 2-CTA thread-block clusters.
#include <cooperative_groups.h>

#include "chain_common.cuh"

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
  macc *Gt = const_cast<macc *>(a.G);
  double acc[4] = {0.0, 0.0, 0.0, 0.0};   // Σ t0 gx0, Σ t1 gx1, Σ z², bad
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    const NodeH h = node_heights(xw[k], xw[N + k], sp.inv_sigma[0], sp.inv_sigma[1], a.z_top, true);
    const size_t t0 = tix(c, 0, k, N), t1 = tix(c, 1, k, N);
    const double G0 = dq_g(Gt[t0]), G1 = dq_g(Gt[t1]);
    Gt[t0] = 0;
    Gt[t1] = 0;
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
    double lp = dq_ll(a.ll[c]);
    if (a.prior_on)
      lp += -0.5 * acc[2] - N * log(2.0 * M_PI) + log(sp.r[0]) + log1p(-sp.r[0]) + log(sp.r[1]) + log1p(-sp.r[1]);
    a.ll[c] = 0;
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
  const macc *Gt = a.G;
  double acc[2] = {0.0, 0.0};   // Σ t_l gx_l, Σ z_l²
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    const NodeH h = node_heights(xw[k], xw[N + k], sp.inv_sigma[0], sp.inv_sigma[1], a.z_top, true);
    const double G0 = dq_g(Gt[tix(c, 0, k, N)]), G1 = dq_g(Gt[tix(c, 1, k, N)]);
    const double g = l == 0 ? G0 * h.J0 + G1 * h.J10 : G1 * h.J11;
    gx[k] = g;
    acc[0] += (l == 0 ? h.t0 : h.t1) * g;
    const double zv = vc[l * N + k];
    acc[1] += zv * zv;
  }
  block_sum<2>(acc);
  cluster.sync();   // both CTAs have read ∂ℓ/∂H: clear it (CTA l its surface)
  macc *Gw = const_cast<macc *>(a.G);
  for (int k = threadIdx.x; k < N; k += blockDim.x) Gw[tix(c, l, k, N)] = 0;
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
    double lp = dq_ll(a.ll[c]);
    if (a.prior_on)
      lp += -0.5 * (part[0] + o[0]) - N * log(2.0 * M_PI) + log(sp.r[0]) + log1p(-sp.r[0]) + log(sp.r[1]) +
            log1p(-sp.r[1]);
    a.ll[c] = 0;
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

// dynamic shared memory of the non-centred kernels: 4N doubles of DFT work + twiddles
// (K3 adds 2N for ∂ll/∂x): up to 200 KiB at N = 4096, so opt in once
// The shared-memory opt-in is per device: set it once per device of the problem.  A
// failure is not recorded as done, so the launch that needs it fails and the caller's
// cudaGetLastError reports it.
static size_t ncp_smem(const mt_problem *p) {
  static bool attr[64] = {false};
  const int d = p->device & 63;
  if (!attr[d]) {
    const int mx = (6 * MT_MAX_NODES + 4 * MT_MAX_AXIS) * (int)sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(k_ncp_heights, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_ncp_finish, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_ncp_heights_cl, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_ncp_finish_cl, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    attr[d] = e == cudaSuccess;
  }
  return (size_t)(4 * p->N + 4 * MT_MAX_AXIS) * sizeof(double);
}

#ifndef MT_NCP_CLUSTER
#define MT_NCP_CLUSTER 1
#endif
void launch_ncp_heights(mt_problem *p, const FinishArgs &a, int C, const float *x, cudaStream_t s) {
  if (MT_NCP_CLUSTER)
    k_ncp_heights_cl<<<dim3(C, 2), MT_THREADS, ncp_smem(p) + (size_t)p->N * sizeof(double), s>>>(a, x);
  else
    k_ncp_heights<<<C, MT_THREADS, ncp_smem(p), s>>>(a, x);
}


void launch_ncp_finish(mt_problem *p, const FinishArgs &a, int C, cudaStream_t s) {
  if (MT_NCP_CLUSTER)
    k_ncp_finish_cl<<<dim3(C, 2), MT_THREADS, ncp_smem(p) + (size_t)p->N * sizeof(double), s>>>(a);
  else
    k_ncp_finish<<<C, MT_THREADS, ncp_smem(p) + (size_t)2 * p->N * sizeof(double), s>>>(a);
}

void launch_ncp_kick(mt_problem *p, int mode, const FinishArgs &a, int C, cudaStream_t s) {
  if (mode == KICK_HALF_DRIFT) k_ncp_kick<KICK_HALF_DRIFT><<<C, MT_THREADS, 0, s>>>(a);
  else if (mode == KICK_FULL_DRIFT) k_ncp_kick<KICK_FULL_DRIFT><<<C, MT_THREADS, 0, s>>>(a);
  else k_ncp_kick<KICK_HALF_LAST><<<C, MT_THREADS, 0, s>>>(a);
  if (mode != KICK_HALF_LAST) launch_ncp_heights(p, a, C, a.x, s);
}
