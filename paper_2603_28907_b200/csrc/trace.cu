// trace.cu — K2: ray x chain trace through the bilinear height fields, fused
// opacity -> flux -> Poisson log-likelihood epilogue and adjoint scatter of
// ∂ℓ/∂H into per-chain shared-memory gradient tiles (B200, sm_100a).
//
// Method: opacity O = ∫ρ du along the sensor ray with the
// Heaviside layer map evaluated exactly on bilinear surfaces (R1,
// R2); λ = w exp(-O/Λ) (R9); Poisson likelihood.
// Gradient: reverse mode by hand: a crossing of surface l at
// (u_c, v_c) with slope g' contributes φ_node(u_c, v_c)/|g'| to ∂B_l/∂h_node.
//
// Mapping: grid = (ray chunks, chain groups of K); block of
// 256 threads; thread = one ray at a time, processing the K chains of its block
// in turn.  The K chains' height fields and gradient tiles live in shared
// memory; ray descriptors are two coalesced float4 loads per ray, shared by
// the K chains; the exact traversal start (DDA state at the band entry) is
// computed once per ray and reused by the K chains.
#include <math.h>

#include "mt_internal.cuh"

namespace {

constexpr int MAXREC = 4;       // crossing records kept in registers per chain x ray
constexpr float GTHR = 0.1f;    // |g'| below which a crossing is re-solved in fp64
constexpr float ZTHR = 1e-3f;   // near-tangent band (m) re-solved in fp64

// sign(a*b - c*d) for a, c >= 0 and b, d > 0, EXACTLY: operands are fp32 values
// with <= 24 significant bits, so the products are exact in fp64.  A filtered
// fp32 test decides all but near-ties (HP3).
__device__ __forceinline__ int cmp_prod(float a, float b, float c, float d) {
  float p = __fmul_rn(a, b), q = __fmul_rn(c, d);
  float diff = __fsub_rn(p, q), tol = __fmul_rn(__fadd_rn(p, q), 1.2e-7f);
  if (diff > tol) return 1;
  if (diff < -tol) return -1;
  double pd = (double)a * (double)b, qd = (double)c * (double)d;
  return (pd > qd) - (pd < qd);
}

struct Ray {
  float ox, oy, dx, dy, dz, s_exit, tb, cnt;
  float adx, ady, iadx, iady;
  int sx, sy;
};

__device__ __forceinline__ Ray load_ray(const float4 *__restrict__ A, const float4 *__restrict__ B,
                                        int64_t r) {
  float4 a = __ldg(A + r), b = __ldg(B + r);
  Ray y;
  y.ox = a.x; y.oy = a.y; y.dx = a.z; y.dy = a.w;
  y.dz = b.x; y.s_exit = b.y; y.tb = b.z; y.cnt = b.w;
  y.adx = fabsf(y.dx); y.ady = fabsf(y.dy);
  y.iadx = y.adx > 0.f ? 1.f / y.adx : 0.f;
  y.iady = y.ady > 0.f ? 1.f / y.ady : 0.f;
  y.sx = y.dx > 0.f ? 1 : (y.dx < 0.f ? -1 : 0);
  y.sy = y.dy > 0.f ? 1 : (y.dy < 0.f ? -1 : 0);
  return y;
}

// Next traversal event of the ray in cell (i, j): bit 1 = crosses an x-line,
// bit 2 = a y-line, bit 4 = leaves the box (top, or a wall line).  Events are
// ordered by exact comparisons; ties step both indices (R16).  s_ev = parameter
// of the event (fp32).  Shared by the hot kernel and the debug export.
__device__ __forceinline__ int dda_next(const Ray &r, int i, int j, const float *Xs,
                                        const float *Ys, int nx, int ny, float z_top,
                                        float &s_ev) {
  float bn = z_top, bd = r.dz;  // top exit z_top/d_z (detectors at z = 0)
  float numx = 0.f, numy = 0.f;
  int ev = 4;
  if (r.sx) {
    numx = r.sx > 0 ? Xs[i + 1] - r.ox : r.ox - Xs[i];  // exact (HP3)
    int c = cmp_prod(numx, bd, bn, r.adx);               // numx/adx vs bn/bd
    if (c < 0) { bn = numx; bd = r.adx; ev = 1; }
    else if (c == 0) ev |= 1;
  }
  if (r.sy) {
    numy = r.sy > 0 ? Ys[j + 1] - r.oy : r.oy - Ys[j];
    int c = cmp_prod(numy, bd, bn, r.ady);
    if (c < 0) { ev = 2; }
    else if (c == 0) ev |= 2;
  }
  if (ev & 4) s_ev = r.s_exit;
  else if (ev & 1) s_ev = numx * r.iadx;
  else s_ev = numy * r.iady;
  if ((ev & 1) && ((r.sx > 0 && i + 1 == nx - 1) || (r.sx < 0 && i == 0))) ev |= 4;
  if ((ev & 2) && ((r.sy > 0 && j + 1 == ny - 1) || (r.sy < 0 && j == 0))) ev |= 4;
  return ev;
}

// Cell index along one axis at ray parameter s: the largest i in [0, n-2]
// with X_i <= x(s) (d >= 0) or X_i < x(s) (d < 0), i.e. the cell the ray is in
// (entering side on ties, R16).  Exact predicate in fp64.
__device__ __forceinline__ int locate_axis(const float *Xs, int n, float o, float d, float s,
                                           float x0, float inv_mean) {
  float xs = fmaf(s, d, o);
  int i = (int)floorf((xs - x0) * inv_mean);
  i = max(0, min(n - 2, i));
  double sd = (double)s * (double)d;
  auto reached = [&](int k) -> bool {
    double dxk = (double)(Xs[k] - o);
    return d < 0.f ? (dxk < sd) : (dxk <= sd);
  };
  while (i < n - 2 && reached(i + 1)) i++;
  while (i > 0 && !reached(i)) i--;
  return i;
}

struct Rec {
  int cell;       // (l << 16) | (i*ny + j)
  float u, v, ig; // crossing position in the cell, 1/|g'|
};

// Below-surface length of the ray inside one cell of one surface and the
// crossings (sign changes of g), in precision T.  g(τ) = g0 + g1 τ + g2 τ².
template <typename T>
struct CellSol {
  T below;
  int n;
  T tc[2], gp[2];
};

template <typename T>
__device__ __forceinline__ CellSol<T> solve_roots(T g0, T g1, T g2, T L) {
  CellSol<T> o;
  o.n = 0;
  T rt[2];
  int nr = 0;
  T disc = g1 * g1 - T(4) * g2 * g0;
  if (g2 == T(0)) {
    if (g1 != T(0)) {
      T t = -g0 / g1;
      if (t > T(0) && t < L) rt[nr++] = t;
    }
  } else if (disc > T(0)) {
    T sq = sqrt(disc);
    T q = T(-0.5) * (g1 + (g1 >= T(0) ? sq : -sq));
    T t1 = q / g2, t2 = g0 / q;
    if (t1 > t2) { T tmp = t1; t1 = t2; t2 = tmp; }
    if (t1 > T(0) && t1 < L) rt[nr++] = t1;
    if (t2 > T(0) && t2 < L && t2 != t1) rt[nr++] = t2;
  }
  // split [0, L] at the roots; sign of g at piece midpoints (strict >, R17)
  T below = T(0);
  T e0 = T(0);
  int prev = 0;
  for (int k = 0; k <= nr; k++) {
    T e1 = k < nr ? rt[k] : L;
    T tm = T(0.5) * (e0 + e1);
    T gm = g0 + tm * (g1 + tm * g2);
    int sg = gm > T(0) ? 1 : -1;
    if (sg > 0) below += e1 - e0;
    if (k > 0 && sg != prev) {
      o.tc[o.n] = e0;
      o.gp[o.n] = g1 + T(2) * g2 * e0;
      o.n++;
    }
    prev = sg;
    e0 = e1;
  }
  o.below = below;
  return o;
}

// Cell-local quadratic g(τ) = h(u(τ), v(τ)) - z(τ), τ = s' - s (R2): with
// h = a + b u + c v + e u v, u = u0 + α τ, v = v0 + β τ, z = d_z (s + τ).
__device__ __forceinline__ void cell_coeffs(float h00, float h10, float h01, float h11, float Xi,
                                            float Yj, float idx, float idy, const Ray &r, float s,
                                            float &u0, float &v0, float &al, float &be, float &g0,
                                            float &g1, float &g2) {
  u0 = (fmaf(s, r.dx, r.ox) - Xi) * idx;
  v0 = (fmaf(s, r.dy, r.oy) - Yj) * idy;
  float z0 = s * r.dz;
  al = r.dx * idx;
  be = r.dy * idy;
  float b = h10 - h00, c = h01 - h00, e = (h11 - h10) - (h01 - h00);
  g0 = (h00 - z0) + u0 * (b + e * v0) + c * v0;
  g1 = b * al + c * be + e * (u0 * be + v0 * al) - r.dz;
  g2 = e * al * be;
}

// fp64 re-solve: coefficients from the exact cell spacing.
__device__ __noinline__ CellSol<double> solve_cell_f64(float h00, float h10, float h01, float h11,
                                                       float Xi, float Xi1, float Yj, float Yj1,
                                                       const Ray &r, float s, float s1,
                                                       double &u0, double &v0, double &al,
                                                       double &be) {
  double ix = 1.0 / ((double)Xi1 - (double)Xi), iy = 1.0 / ((double)Yj1 - (double)Yj);
  u0 = ((double)r.ox + (double)s * (double)r.dx - (double)Xi) * ix;
  v0 = ((double)r.oy + (double)s * (double)r.dy - (double)Yj) * iy;
  double z0 = (double)s * (double)r.dz;
  al = (double)r.dx * ix;
  be = (double)r.dy * iy;
  double b = (double)h10 - h00, c = (double)h01 - h00, e = ((double)h11 - h10) - ((double)h01 - h00);
  double g0 = ((double)h00 - z0) + u0 * (b + e * v0) + c * v0;
  double g1 = b * al + c * be + e * (u0 * be + v0 * al) - (double)r.dz;
  double g2 = e * al * be;
  return solve_roots<double>(g0, g1, g2, (double)s1 - (double)s);
}

struct Geo {
  const float *Xs, *Ys, *idx, *idy;
  int nx, ny, N;
  float z_top;
};

// Process one cell [s, s1] of surface l for one chain: adds the below length
// to B; records (or, SCAT, scatters with factor f) the crossings.
template <bool SCAT>
__device__ __forceinline__ void do_cell(const Geo &g, const Ray &r, const float *Hl, float *Gl,
                                        int l, int i, int j, float s, float s1, float zmin,
                                        float zmax, float &B, Rec *rec, int &nrec, bool &ovf,
                                        float f) {
  float za = s * r.dz, zb = s1 * r.dz;
  if (zb <= zmin) { B += s1 - s; return; }     // whole cell below the surface's lowest node
  if (za >= zmax) return;                       // whole cell above its highest node
  int base = i * g.ny + j;
  float h00 = Hl[base], h10 = Hl[base + g.ny], h01 = Hl[base + 1], h11 = Hl[base + g.ny + 1];
  float cmin = fminf(fminf(h00, h10), fminf(h01, h11));
  float cmax = fmaxf(fmaxf(h00, h10), fmaxf(h01, h11));
  if (zb <= cmin) { B += s1 - s; return; }     // bilinear min is at a corner
  if (za >= cmax) return;
  float u0, v0, al, be, g0, g1, g2;
  cell_coeffs(h00, h10, h01, h11, g.Xs[i], g.Ys[j], g.idx[i], g.idy[j], r, s, u0, v0, al,
                     be, g0, g1, g2);
  float L = s1 - s;
  CellSol<float> so = solve_roots<float>(g0, g1, g2, L);
  bool bad = false;
  for (int k = 0; k < so.n; k++) bad |= fabsf(so.gp[k]) < GTHR;
  if (!bad && g2 != 0.f) {  // near-tangent: vertex inside with |g(vertex)| small
    float tv = -g1 / (2.f * g2);
    float disc = g1 * g1 - 4.f * g2 * g0;
    if (tv > 0.f && tv < L && fabsf(disc) < 4.f * fabsf(g2) * ZTHR) bad = true;
  }
  float below;
  int ncr;
  float uc[2], vc[2], igc[2];
  if (!bad) {
    below = so.below;
    ncr = so.n;
    for (int k = 0; k < 2; k++) {
      if (k < ncr) {
        uc[k] = u0 + al * so.tc[k];
        vc[k] = v0 + be * so.tc[k];
        igc[k] = 1.f / fabsf(so.gp[k]);
      }
    }
  } else {
    double du0, dv0, dal, dbe;
    CellSol<double> sd = solve_cell_f64(h00, h10, h01, h11, g.Xs[i], g.Xs[i + 1], g.Ys[j],
                                        g.Ys[j + 1], r, s, s1, du0, dv0, dal, dbe);
    below = (float)sd.below;
    ncr = sd.n;
    for (int k = 0; k < 2; k++) {
      if (k < ncr) {
        uc[k] = (float)(du0 + dal * sd.tc[k]);
        vc[k] = (float)(dv0 + dbe * sd.tc[k]);
        igc[k] = (float)(1.0 / fabs(sd.gp[k]));
      }
    }
  }
  B += below;
  for (int k = 0; k < 2; k++) {
    if (k < ncr) {
      if (SCAT) {
        float w = f * igc[k], u = uc[k], v = vc[k];
        atomicAdd(Gl + base, w * (1.f - u) * (1.f - v));
        atomicAdd(Gl + base + g.ny, w * u * (1.f - v));
        atomicAdd(Gl + base + 1, w * (1.f - u) * v);
        atomicAdd(Gl + base + g.ny + 1, w * u * v);
      } else {
        Rec rc;
        rc.cell = (l << 16) | base;
        rc.u = uc[k]; rc.v = vc[k]; rc.ig = igc[k];
#pragma unroll
        for (int m = 0; m < MAXREC; m++)
          if (m == nrec) rec[m] = rc;
        if (nrec < MAXREC) nrec++;
        else ovf = true;
      }
    }
  }
}

// Walk the cells of the band [s0, s_hi] for one chain from DDA state (i0, j0).
template <bool SCAT>
__device__ __forceinline__ void walk(const Geo &g, const Ray &r, int i0, int j0, float s0,
                                     float s_hi, const float *Hk, float *Gk, float4 bd, float &B0,
                                     float &B1, Rec *rec, int &nrec, bool &ovf, float f0,
                                     float f1) {
  int i = i0, j = j0;
  float s = s0;
  for (int guard = 0; guard < 4 * (MT_MAX_AXIS + 2); guard++) {
    float s_ev;
    int ev = dda_next(r, i, j, g.Xs, g.Ys, g.nx, g.ny, g.z_top, s_ev);
    float s1 = fminf(s_ev, r.s_exit);
    if (s1 > s) {
      do_cell<SCAT>(g, r, Hk, Gk, 0, i, j, s, s1, bd.x, bd.y, B0, rec, nrec, ovf, f0);
      do_cell<SCAT>(g, r, Hk + g.N, Gk + g.N, 1, i, j, s, s1, bd.z, bd.w, B1, rec, nrec, ovf, f1);
    }
    if ((ev & 4) || s1 >= s_hi) break;
    if (ev & 1) i += r.sx;
    if (ev & 2) j += r.sy;
    s = s1;
  }
}

}  // namespace

template <int K, int MODE>
__global__ void __launch_bounds__(MT_THREADS) k_trace(TraceArgs a) {
  extern __shared__ __align__(16) float smem[];
  const int nx = a.tc.nx, ny = a.tc.ny, N = a.tc.N;
  float *Xs = smem, *Ys = Xs + nx, *idx = Ys + ny, *idy = idx + nx;
  int geo_words = (2 * nx + 2 * ny + 3) & ~3;
  float *Hs = smem + geo_words;                       // [K][2N]
  float *Gs = Hs + K * 2 * N;                         // [K][2N] (TRACE_LL)
  __shared__ double red[MT_THREADS / 32][K];

  const int tid = threadIdx.x;
  const int c0 = blockIdx.y * K;
  const int nk = min(K, a.C - c0);
  for (int k = tid; k < nx; k += blockDim.x) {
    Xs[k] = a.X[k];
    idx[k] = k < nx - 1 ? 1.f / (a.X[k + 1] - a.X[k]) : 0.f;
  }
  for (int k = tid; k < ny; k += blockDim.x) {
    Ys[k] = a.Y[k];
    idy[k] = k < ny - 1 ? 1.f / (a.Y[k + 1] - a.Y[k]) : 0.f;
  }
  {
    const float *src = a.H + (size_t)c0 * 2 * N;
    const int nh = nk * 2 * N;
    if ((N & 1) == 0) {  // 2N % 4 == 0: float4 path (rows stay 16-B aligned)
      const float4 *s4 = reinterpret_cast<const float4 *>(src);
      float4 *d4 = reinterpret_cast<float4 *>(Hs);
      for (int k = tid; k < nh / 4; k += blockDim.x) d4[k] = __ldg(s4 + k);
    } else {
      for (int k = tid; k < nh; k += blockDim.x) Hs[k] = __ldg(src + k);
    }
    if (MODE == TRACE_LL)
      for (int k = tid; k < K * 2 * N; k += blockDim.x) Gs[k] = 0.f;
  }
  __shared__ float4 bds[K];
  __shared__ float llacc[K][MT_THREADS];
  if (tid < K) bds[tid] = tid < nk ? a.band[c0 + tid] : make_float4(0.f, 0.f, 0.f, 0.f);
  for (int k = 0; k < K; k++) llacc[k][tid] = 0.f;
  __syncthreads();
  float zlo = 3.0e38f;
  for (int k = 0; k < nk; k++) zlo = fminf(zlo, bds[k].x);

  Geo g;
  g.Xs = Xs; g.Ys = Ys; g.idx = idx; g.idy = idy; g.nx = nx; g.ny = ny; g.N = N;
  g.z_top = a.tc.z_top;
  const float x0 = Xs[0], y0 = Ys[0];
  const float inv_mx = (float)(nx - 1) / (Xs[nx - 1] - Xs[0]);
  const float inv_my = (float)(ny - 1) / (Ys[ny - 1] - Ys[0]);

  const int64_t r_begin = (int64_t)blockIdx.x * a.rays_per_block;
  const int64_t r_end = min(a.R, r_begin + a.rays_per_block);
  for (int64_t rr = r_begin + tid; rr < r_end; rr += blockDim.x) {
    Ray r = load_ray(a.ray_a, a.ray_b, rr);
    // union band of the block's chains: the ray is below every surface before s_lo
    float s_lo = fminf(zlo / r.dz, r.s_exit);
    bool walkable = s_lo < r.s_exit;
    int i0 = 0, j0 = 0;
    if (walkable) {
      i0 = locate_axis(Xs, nx, r.ox, r.dx, s_lo, x0, inv_mx);
      j0 = locate_axis(Ys, ny, r.oy, r.dy, s_lo, y0, inv_my);
    }
#pragma unroll 1
    for (int k = 0; k < nk; k++) {
      const float *Hk = Hs + k * 2 * N;
      float *Gk = Gs + k * 2 * N;
      const float4 bd = bds[k];
      float B0 = s_lo, B1 = s_lo;
      Rec rec[MAXREC];
      int nrec = 0;
      bool ovf = false;
      float s_hi = fminf(bd.w / r.dz, r.s_exit);
      if (walkable)
        walk<false>(g, r, i0, j0, s_lo, s_hi, Hk, Gk, bd, B0, B1, rec, nrec, ovf, 0.f, 0.f);
      if (MODE == TRACE_LL) {
        // fused epilogue: t = ln(λ/C) (C > 0) or ln λ (C = 0)  (HP4, R15)
        float t = r.tb - (a.tc.k0 * B0 + a.tc.k1 * B1) * a.tc.inv_att;
        float ll, dldO;
        if (r.cnt > 0.f) {
          float em1 = expm1f(t);
          ll = -r.cnt * (em1 - t);
          dldO = r.cnt * em1 * a.tc.inv_att;      // (λ - C)/Λ
        } else {
          float lam = expf(t);
          ll = -lam;
          dldO = lam * a.tc.inv_att;
        }
        llacc[k][tid] += ll;
        float f0 = dldO * a.tc.k0, f1 = dldO * a.tc.k1;
        if (!ovf) {
#pragma unroll
          for (int m = 0; m < MAXREC; m++) {
            if (m < nrec) {
              Rec rc = rec[m];
              int l = rc.cell >> 16, base = rc.cell & 0xffff;
              float w = (l ? f1 : f0) * rc.ig, u = rc.u, v = rc.v;
              float *Gl = Gk + l * N;
              atomicAdd(Gl + base, w * (1.f - u) * (1.f - v));
              atomicAdd(Gl + base + ny, w * u * (1.f - v));
              atomicAdd(Gl + base + 1, w * (1.f - u) * v);
              atomicAdd(Gl + base + ny + 1, w * u * v);
            }
          }
        } else {  // rare: more crossings than registers hold -> scattering re-walk
          float d0 = 0.f, d1 = 0.f;
          int dn = 0;
          bool dov = false;
          walk<true>(g, r, i0, j0, s_lo, s_hi, Hk, Gk, bd, d0, d1, rec, dn, dov, f0, f1);
        }
      } else {
        int64_t o = (int64_t)(c0 + k) * a.R + rr;
        a.Lout[3 * o + 0] = B0;
        a.Lout[3 * o + 1] = B1 - B0;
        a.Lout[3 * o + 2] = r.s_exit - B1;
        a.Oout[o] = a.tc.k0 * B0 + a.tc.k1 * B1 + a.obase[rr];
      }
    }
  }

  if (MODE == TRACE_LL) {
    const int lane = tid & 31, wid = tid >> 5;
    for (int k = 0; k < nk; k++) {
      float v = llacc[k][tid];
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) red[wid][k] = (double)v;
    }
    __syncthreads();
    if (tid < nk) {
      double s = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); w++) s += red[w][tid];
      atomicAdd(a.ll + c0 + tid, s);
    }
    for (int k = tid; k < nk * 2 * N; k += blockDim.x) {
      float v = Gs[k];
      if (v != 0.f) atomicAdd(a.G + (size_t)c0 * 2 * N + k, v);
    }
  }
}

// ---------------------------------------------------------------------------
// debug traversal: the exact DDA from s = 0 with the same device functions
// ---------------------------------------------------------------------------
__global__ void k_debug_traversal(TraceArgs a, int64_t ray, int32_t *ij, float *si, float *so,
                                  int cap, int32_t *n_out) {
  __shared__ float Xs[MT_MAX_AXIS], Ys[MT_MAX_AXIS];
  const int nx = a.tc.nx, ny = a.tc.ny;
  for (int k = threadIdx.x; k < nx; k += blockDim.x) Xs[k] = a.X[k];
  for (int k = threadIdx.x; k < ny; k += blockDim.x) Ys[k] = a.Y[k];
  __syncthreads();
  if (threadIdx.x) return;
  Ray r = load_ray(a.ray_a, a.ray_b, ray);
  const float inv_mx = (float)(nx - 1) / (Xs[nx - 1] - Xs[0]);
  const float inv_my = (float)(ny - 1) / (Ys[ny - 1] - Ys[0]);
  int i = locate_axis(Xs, nx, r.ox, r.dx, 0.f, Xs[0], inv_mx);
  int j = locate_axis(Ys, ny, r.oy, r.dy, 0.f, Ys[0], inv_my);
  float s = 0.f;
  int n = 0;
  for (int guard = 0; guard < 4 * (MT_MAX_AXIS + 2); guard++) {
    float s_ev;
    int ev = dda_next(r, i, j, Xs, Ys, nx, ny, a.tc.z_top, s_ev);
    float s1 = fminf(s_ev, r.s_exit);
    if (n < cap) { ij[2 * n] = i; ij[2 * n + 1] = j; si[n] = s; so[n] = s1; }
    n++;
    if (ev & 4) break;
    if (ev & 1) i += r.sx;
    if (ev & 2) j += r.sy;
    s = s1;
  }
  *n_out = n;
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
template <int K, int MODE>
static cudaError_t launch_k(const TraceArgs &a, dim3 grid, size_t smem, cudaStream_t s) {
  static size_t smem_set[16] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (smem > 48 * 1024 && smem_set[dev & 15] < smem) {
    cudaError_t e = cudaFuncSetAttribute(k_trace<K, MODE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    smem_set[dev & 15] = smem;
  }
  k_trace<K, MODE><<<grid, MT_THREADS, smem, s>>>(a);
  return cudaGetLastError();
}

static int pick_k(const mt_problem *p, int C) {
  if (p->trace_k > 0) return p->trace_k;
  size_t per_chain = (size_t)16 * p->N;   // H + G tiles, fp32
  int k = 8;
  while (k > 1 && (size_t)k * per_chain > 40 * 1024) k >>= 1;
  while (k > 1 && (C + k - 1) / k < p->num_sms) k >>= 1;
  return k;
}

cudaError_t launch_trace(mt_problem *p, int mode, int C, const float *H, const float4 *band,
                         float *G, double *ll, float *L, float *O, cudaStream_t s) {
  if (C <= 0 || p->R <= 0) return cudaSuccess;
  TraceArgs a;
  a.tc = p->tc;
  a.X = p->d_X; a.Y = p->d_Y;
  a.ray_a = p->d_ray_a; a.ray_b = p->d_ray_b; a.obase = p->d_obase;
  a.R = p->R;
  a.C = C;
  a.H = H; a.band = band; a.G = G; a.ll = ll; a.Lout = L; a.Oout = O;
  int K = pick_k(p, C);
  int groups = (C + K - 1) / K;
  int64_t S;
  if (p->trace_s > 0) S = p->trace_s;
  else {
    int64_t target = (int64_t)p->num_sms * 8;  // ~8 resident-block slots per SM
    S = (target + groups - 1) / groups;
    int64_t max_s = (p->R + MT_THREADS - 1) / MT_THREADS;
    if (S > max_s) S = max_s;
    if (S < 1) S = 1;
  }
  a.rays_per_block = (p->R + S - 1) / S;
  S = (p->R + a.rays_per_block - 1) / a.rays_per_block;
  dim3 grid((unsigned)S, (unsigned)groups);
  int geo_words = (2 * p->nx + 2 * p->ny + 3) & ~3;
  size_t smem = (size_t)4 * (geo_words + (size_t)K * 2 * p->N * (mode == TRACE_LL ? 2 : 1));
  cudaError_t e = cudaSuccess;
  bool rec = p->timing && p->n_rec < (int)p->ev_a.size();
  if (rec) cudaEventRecord(p->ev_a[p->n_rec], s);
#define MT_DISPATCH(KK)                                                         \
  case KK:                                                                      \
    e = mode == TRACE_LL ? launch_k<KK, TRACE_LL>(a, grid, smem, s)          \
                         : launch_k<KK, TRACE_PATH>(a, grid, smem, s);       \
    break;
  switch (K) {
    MT_DISPATCH(1)
    MT_DISPATCH(2)
    MT_DISPATCH(4)
    MT_DISPATCH(8)
    default: return cudaErrorInvalidValue;
  }
#undef MT_DISPATCH
  if (rec) { cudaEventRecord(p->ev_b[p->n_rec], s); p->n_rec++; }
  p->all_launches++;
  p->trace_launches++;
  p->pairs += (double)C * (double)p->R;
  return e;
}

cudaError_t launch_debug_traversal(mt_problem *p, int64_t ray, int32_t *d_ij, float *d_si,
                                   float *d_so, int cap, int32_t *d_n) {
  TraceArgs a;
  a.tc = p->tc;
  a.X = p->d_X; a.Y = p->d_Y;
  a.ray_a = p->d_ray_a; a.ray_b = p->d_ray_b;
  k_debug_traversal<<<1, 128>>>(a, ray, d_ij, d_si, d_so, cap, d_n);
  p->all_launches++;
  return cudaGetLastError();
}
