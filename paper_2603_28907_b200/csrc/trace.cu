// trace.cu — K2: ray x chain trace through the bilinear height fields, fused
// opacity -> flux -> Poisson log-likelihood epilogue and adjoint scatter of
// ∂ℓ/∂H (B200, sm_100a).
//
// Method: opacity O = ∫ρ du along the sensor ray with the
// Heaviside layer map evaluated exactly on bilinear surfaces (R1,
// R2); λ = w exp(-O/Λ) (R9); Poisson likelihood.
// Gradient: reverse mode by hand: a crossing of surface l at
// (u_c, v_c) with slope g' contributes φ_node(u_c, v_c)/|g'| to ∂B_l/∂h_node.
//
// The traversal (ordered cells of each ray, a2) does not depend on the
// geometry, so it is computed ONCE per problem by k_build_trav with exact
// predicates (HP3) and stored as a CSR list; the hot kernels only read it.
//
// Two mappings:
//  * chain lanes (C >= 16, the hot configuration): warp = one ray x 32 chains,
//    lane = chain.  Ray, traversal and control flow are warp-uniform; heights
//    are coalesced 128-B lines of the chain-interleaved layout (shared memory
//    when a 32-chain tile fits, else L1-cached global loads); the adjoint is a
//    coalesced RED.ADD.F32 into the interleaved ∂ℓ/∂H buffer (no CAS loops, no
//    intra-warp contention).
//  * ray lanes (small C, e.g. the single-chain ray-sharded config): block = K
//    chains with shared-memory height and gradient tiles, thread = ray.
#include <cuda_fp16.h>
#include <math.h>
#include <string.h>

#include <algorithm>

#include "mt_internal.cuh"

namespace {

#ifndef MT_GTHR
#define MT_GTHR 0.05f
#endif
#ifndef MT_ZTHR
#define MT_ZTHR 1e-4f
#endif
constexpr float GTHR = MT_GTHR;   // |g'| below which a crossing is re-solved in fp64
constexpr float ZTHR = MT_ZTHR;   // near-tangent band (m) re-solved in fp64

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
};

__device__ __forceinline__ Ray load_ray(const float4 *__restrict__ A, const float4 *__restrict__ B,
                                        int64_t r) {
  float4 a = __ldg(A + r), b = __ldg(B + r);
  Ray y;
  y.ox = a.x; y.oy = a.y; y.dx = a.z; y.dy = a.w;
  y.dz = b.x; y.s_exit = b.y; y.tb = b.z; y.cnt = b.w;
  return y;
}

// ---------------------------------------------------------------------------
// exact traversal (a2): used only by the per-problem builder
// ---------------------------------------------------------------------------
struct DdaRay {
  Ray r;
  float adx, ady, iadx, iady;
  int sx, sy;
};

__device__ __forceinline__ DdaRay dda_ray(const Ray &r) {
  DdaRay y;
  y.r = r;
  y.adx = fabsf(r.dx); y.ady = fabsf(r.dy);
  y.iadx = y.adx > 0.f ? 1.f / y.adx : 0.f;
  y.iady = y.ady > 0.f ? 1.f / y.ady : 0.f;
  y.sx = r.dx > 0.f ? 1 : (r.dx < 0.f ? -1 : 0);
  y.sy = r.dy > 0.f ? 1 : (r.dy < 0.f ? -1 : 0);
  return y;
}

// Next event of the ray in cell (i, j): bit 1 = crosses an x-line, bit 2 = a
// y-line, bit 4 = leaves the box (top, or a wall line).  Events are ordered by
// exact comparisons; ties step both indices (R16).  s_ev = event parameter.
__device__ __forceinline__ int dda_next(const DdaRay &q, int i, int j, const float *Xs,
                                        const float *Ys, int nx, int ny, float z_top,
                                        float &s_ev, int *fcode = nullptr) {
  float bn = z_top, bd = q.r.dz;  // top exit z_top/d_z (detectors at z = 0)
  float numx = 0.f, numy = 0.f;
  int ev = 4;
  if (q.sx) {
    numx = q.sx > 0 ? Xs[i + 1] - q.r.ox : q.r.ox - Xs[i];  // exact (HP3)
    int c = cmp_prod(numx, bd, bn, q.adx);                   // numx/adx vs bn/bd
    if (c < 0) { bn = numx; bd = q.adx; ev = 1; }
    else if (c == 0) ev |= 1;
  }
  if (q.sy) {
    numy = q.sy > 0 ? Ys[j + 1] - q.r.oy : q.r.oy - Ys[j];
    int c = cmp_prod(numy, bd, bn, q.ady);
    if (c < 0) { ev = 2; }
    else if (c == 0) ev |= 2;
  }
  if (ev & 4) s_ev = q.r.s_exit;
  else if (ev & 1) s_ev = numx * q.iadx;
  else s_ev = numy * q.iady;
  if (fcode) *fcode = (ev & 4) ? 0 : (ev & 3);   // which formula gave s_ev (ray-lane step codes)
  if ((ev & 1) && ((q.sx > 0 && i + 1 == nx - 1) || (q.sx < 0 && i == 0))) ev |= 4;
  if ((ev & 2) && ((q.sy > 0 && j + 1 == ny - 1) || (q.sy < 0 && j == 0))) ev |= 4;
  return ev;
}

// Cell index along one axis at the ray origin: the largest i in [0, n-2] with
// X_i <= o (d >= 0) or X_i < o (d < 0), i.e. the cell in the direction of
// travel when o lies on a line (R16).
__device__ __forceinline__ int start_axis(const float *Xs, int n, float o, float d) {
  int i = 0;
  for (int k = 0; k < n - 1; k++)
    if (d < 0.f ? (Xs[k] < o) : (Xs[k] <= o)) i = k;
  return i;
}

// ---------------------------------------------------------------------------
// per-cell analytic solve (a3)
// ---------------------------------------------------------------------------
template <typename T>
struct CellSol {
  T below;
  int n;
  T tc[2], gp[2];
};

// Split [0, L] at the real roots of g0 + g1 τ + g2 τ² (stable quadratic form;
// g2 = 0 gives the linear root through the second formula) and add the pieces
// with g > 0 at their midpoint (strict, R17); crossings = sign changes.
template <typename T>
__device__ __forceinline__ CellSol<T> classify(T g0, T g1, T g2, T L, T t1, T t2, bool two) {
  CellSol<T> o;
  o.n = 0;
  T rt[2];
  int nr = 0;
  if (two) {
    if (t1 > t2) { T tmp = t1; t1 = t2; t2 = tmp; }
    if (t1 > T(0) && t1 < L) rt[nr++] = t1;
    if (t2 > T(0) && t2 < L && t2 != t1) rt[nr++] = t2;
  }
  T below = T(0), e0 = T(0);
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

// fp64 re-solve of one cell from the same fp32 inputs, exact cell spacing
// (HP2 lever 1), with the oracle-style midpoint classification.  Rare;
// noinline so its double-precision registers stay out of the callers' loops,
// and everything is passed and returned BY VALUE (a reference to a caller's
// accumulator would pin it to local memory).
struct Fix {
  float below;
  int n;
  float u[2], v[2], ig[2];
};

__device__ __noinline__ Fix fix64(double h00, double h10, double h01, double h11, float Xi, float Xi1,
                                  float Yj, float Yj1, Ray r, double s, double s1) {
  const double ix = 1.0 / ((double)Xi1 - (double)Xi), iy = 1.0 / ((double)Yj1 - (double)Yj);
  const double u0 = ((double)r.ox + s * (double)r.dx - (double)Xi) * ix;
  const double v0 = ((double)r.oy + s * (double)r.dy - (double)Yj) * iy;
  const double z0 = s * (double)r.dz;
  const double al = (double)r.dx * ix, be = (double)r.dy * iy;
  const double b = h10 - h00, c = h01 - h00, e = (h11 - h10) - (h01 - h00);
  const double g0 = (h00 - z0) + u0 * (b + e * v0) + c * v0;
  const double g1 = b * al + c * be + e * (u0 * be + v0 * al) - (double)r.dz;
  const double g2 = e * al * be;
  const double L = s1 - s;
  const double disc = g1 * g1 - 4.0 * g2 * g0;
  double t1 = 0, t2 = 0;
  const bool two = disc > 0.0;
  if (two) {
    const double q = -0.5 * (g1 + (g1 >= 0.0 ? sqrt(disc) : -sqrt(disc)));
    t1 = q / g2;   // ±inf when g2 = 0: out of range
    t2 = g0 / q;
  }
  const CellSol<double> sd = classify<double>(g0, g1, g2, L, t1, t2, two);
  Fix x;
  x.below = (float)sd.below;
  x.n = sd.n;
  for (int k = 0; k < 2; k++) {
    x.u[k] = (float)(u0 + al * sd.tc[k]);
    x.v[k] = (float)(v0 + be * sd.tc[k]);
    x.ig[k] = (float)(1.0 / fabs(sd.gp[k]));
  }
  return x;
}

// One surface over one cell piece [s, s1] of a ray, fp32 (a3).  In cell-local
// coordinates u = (x - X_i)/ΔX_i, v = (y - Y_j)/ΔY_j the ray is (u0 + α τ,
// v0 + β τ) for τ ∈ [0, Δs] (cg = {u0, v0, α, β}, from the stored per-cell
// geometry, a0) and the bilinear surface h = a + b u + c v + e u v (R2), so
// g(τ) = h - d_z (s + τ) = g0 + g1 τ + g2 τ².  With g(0) and g(Δs) of
// different sign there is exactly one crossing; with equal signs there are
// two iff the vertex lies inside and g(vertex) = -disc/(4 g2) has the other
// sign.  Adds the below-surface length to B, calls emit(u_c, v_c, 1/|g'|)
// per crossing, and returns false (adding nothing) for an ill-conditioned
// cell: |g'| < GTHR at a crossing or a near-tangent vertex (HP2).
template <class Emit>
__device__ __forceinline__ bool solve32(float h00, float h10, float h01, float h11, float4 cg,
                                        float za, float Ls, float dz, float &B, Emit &&emit) {
  const float u0 = cg.x, v0 = cg.y, al = cg.z, be = cg.w;
  const float b = h10 - h00, c = h01 - h00, e = (h11 - h10) - (h01 - h00);
  const float g0 = (h00 - za) + u0 * (b + e * v0) + c * v0;
  const float g1 = b * al + c * be + e * (u0 * be + v0 * al) - dz;
  const float g2 = e * al * be;
  const float gL = g0 + Ls * (g1 + Ls * g2);
  // |g| < 1 mm where the ray enters or leaves the cell: the surface passes within
  // fp32 rounding of the cell edge, where the bilinear patches meet at a kink; the
  // two cells' fp32 quadratics can then disagree on the sign there and invent (or
  // lose) a crossing pair around a sliver of zero length whose adjoint terms add up.
  // Decide it in fp64 (HP2), like a near-tangent vertex.
  if (fabsf(g0) < ZTHR || fabsf(gL) < ZTHR) return false;
  const float disc = fmaf(g1, g1, -4.f * g2 * g0);
  const bool p0 = g0 > 0.f;
  const float a2 = 2.f * g2;
  const bool vin = -g1 * a2 > 0.f && fabsf(g1) < Ls * fabsf(a2);   // vertex inside (0, Δs)
#ifndef MT_LAZY_ROOTS
#define MT_LAZY_ROOTS 1
#endif
#if MT_LAZY_ROOTS
  // the roots only where a crossing is possible (a no-crossing cell skips RSQ + 2 RCP)
  auto roots = [&](float &ta, float &tb) {
    float q = 0.f;
    if (disc > 0.f) q = -0.5f * (g1 + copysignf(disc * rsqrtf(disc), g1));
    ta = __fdividef(g0, q);
    tb = __fdividef(q, g2);
  };
#else
  float q = 0.f;
  if (disc > 0.f) q = -0.5f * (g1 + copysignf(disc * rsqrtf(disc), g1));
  const float ta0 = __fdividef(g0, q), tb0 = __fdividef(q, g2);       // the two roots (tb = ±inf if g2 = 0)
  auto roots = [&](float &ta, float &tb) { ta = ta0; tb = tb0; };
#endif
  if (p0 != (gL > 0.f)) {                         // exactly one crossing
    float ta, tb;
    roots(ta, tb);
    // the root in [0, Δs]: of the two, the one nearer the interval (rounding
    // can put the true root just outside when it sits at a cell edge)
    const float ca = fminf(fmaxf(ta, 0.f), Ls), cb = fminf(fmaxf(tb, 0.f), Ls);
    const float t = fabsf(ta - ca) <= fabsf(tb - cb) ? ca : cb;
    const float gp = g1 + a2 * t;
    if (fabsf(gp) < GTHR || !(disc > 0.f)) return false;
    B += p0 ? t : Ls - t;
    emit(u0 + al * t, v0 + be * t, __fdividef(1.f, fabsf(gp)));
  } else if (disc > 0.f && vin && ((g2 > 0.f) == p0)) {   // two crossings
    float ta, tb;
    roots(ta, tb);
    const float t1 = fminf(ta, tb), t2 = fmaxf(ta, tb);
    const float gp1 = g1 + a2 * t1, gp2 = g1 + a2 * t2;
    if (fabsf(gp1) < GTHR || fabsf(gp2) < GTHR) return false;
    B += p0 ? Ls - (t2 - t1) : (t2 - t1);
    emit(u0 + al * t1, v0 + be * t1, __fdividef(1.f, fabsf(gp1)));
    emit(u0 + al * t2, v0 + be * t2, __fdividef(1.f, fabsf(gp2)));
  } else {                                        // no crossing
    if (vin && fabsf(disc) < 2.f * fabsf(a2) * ZTHR) return false;   // near-tangent
    if (p0) B += Ls;
  }
  return true;
}

// solve32 with the ray-only parts K = u0 β + v0 α, M = α β stored per cell (a0) and the
// one-crossing root from the cancellation-free form with |g'| = √D (the chain-lanes solve).
template <class Emit>
__device__ __forceinline__ bool solve32k(float h00, float h10, float h01, float h11, float4 cg, float2 km,
                                         float za, float Ls, float dz, float &B, Emit &&emit) {
  const float u0 = cg.x, v0 = cg.y, al = cg.z, be = cg.w;
  const float b = h10 - h00, c = h01 - h00, e = (h11 - h10) - (h01 - h00);
  const float g0 = (h00 - za) + u0 * (b + e * v0) + c * v0;
  const float g1 = fmaf(b, al, fmaf(c, be, fmaf(e, km.x, -dz)));
  const float g2 = e * km.y;
  const float gL = g0 + Ls * (g1 + Ls * g2);
  if (fabsf(g0) < ZTHR || fabsf(gL) < ZTHR) return false;
  const bool p0 = g0 > 0.f, pL = gL > 0.f;
  const float D = fmaf(g1, g1, -4.f * g2 * g0);
  if (p0 != pL) {
    if (!(D >= GTHR * GTHR)) return false;
    const float r = rsqrtf(D), sq = D * r;
    const float ssq = pL ? sq : -sq;
    const bool nc = (g1 > 0.f) == pL;
    const float t = fminf(fmaxf(__fdividef(nc ? -2.f * g0 : ssq - g1, nc ? g1 + ssq : 2.f * g2), 0.f), Ls);
    B += p0 ? t : Ls - t;
    emit(u0 + al * t, v0 + be * t, r);
    return true;
  }
  const float a2 = 2.f * g2;
  const bool vin = -g1 * a2 > 0.f && fabsf(g1) < Ls * fabsf(a2);
  if (vin && D > 0.f && ((g2 > 0.f) == p0)) {
    if (!(D >= GTHR * GTHR)) return false;
    const float r = rsqrtf(D);
    const float q = -0.5f * (g1 + copysignf(D * r, g1));
    const float ta = __fdividef(g0, q), tb = __fdividef(q, g2);
    const float t1 = fminf(ta, tb), t2 = fmaxf(ta, tb);
    B += p0 ? Ls - (t2 - t1) : (t2 - t1);
    emit(u0 + al * t1, v0 + be * t1, r);
    emit(u0 + al * t2, v0 + be * t2, r);
    return true;
  }
  if (vin && fabsf(D) < 2.f * fabsf(a2) * ZTHR) return false;
  if (p0) B += Ls;
  return true;
}

// Stored per-cell geometry {u, v, α, β} is taken at the cell's entry s_in; a
// walk that starts inside the cell (at the band entry s_lo) moves it by
// ds = s_lo - s_in.  For every later cell ds = 0 exactly.
__device__ __forceinline__ float4 shift_geo(float4 cg, float ds) {
  cg.x = fmaf(cg.z, ds, cg.x);
  cg.y = fmaf(cg.w, ds, cg.y);
  return cg;
}

struct Geo {
  const float *Xs, *Ys, *idx, *idy;
  int nx, ny, N;
};

// Node coordinates and inverse spacings, at static shared addresses (indexed
// directly: no pointer registers, no address setup in the hot loops).
__shared__ float sgeo[4][MT_MAX_AXIS];   // X, Y, 1/ΔX, 1/ΔY

// Exact cell boundaries for the fp64 re-solves (HP2/HP3): a crossing within fp32
// rounding of a cell edge must land in the right cell — the two bilinear patches
// meet there with a kink, so the neighbour's |g'| (and hence the adjoint weight)
// would be wrong — so fix64 takes the boundary parameters in fp64 from the exact
// fp32 inputs instead of the stored fp32 s_out.  Boundary between stored cells
// wa -> wb: the x-line (i changed) or y-line the exact DDA crossed.
__device__ __forceinline__ double cell_event64(const Ray &r, int wa, int wb) {
  const int ia = cell_i(wa), ib = cell_i(wb);
  if (ia != ib) return ((double)sgeo[0][ia > ib ? ia : ib] - (double)r.ox) / (double)r.dx;
  const int ja = cell_j(wa), jb = cell_j(wb);
  return ((double)sgeo[1][ja > jb ? ja : jb] - (double)r.oy) / (double)r.dy;
}

// The in-box exit parameter in fp64 (a0: top z_top/d_z or the first side wall).
__device__ __forceinline__ double exit64(const Ray &r, int nx, int ny, float z_top) {
  double s = (double)z_top / (double)r.dz;
  if (r.dx > 0.f) s = fmin(s, ((double)sgeo[0][nx - 1] - (double)r.ox) / (double)r.dx);
  if (r.dx < 0.f) s = fmin(s, ((double)sgeo[0][0] - (double)r.ox) / (double)r.dx);
  if (r.dy > 0.f) s = fmin(s, ((double)sgeo[1][ny - 1] - (double)r.oy) / (double)r.dy);
  if (r.dy < 0.f) s = fmin(s, ((double)sgeo[1][0] - (double)r.oy) / (double)r.dy);
  return s;
}

// fp64 piece [s, s1] of stored cell k of a ray whose stored cells are [kfirst, kend):
// the walk's own start (s_start, not a cell boundary) when k is its first cell,
// else the exact boundaries.
__device__ __forceinline__ void piece64(const TraceArgs &a, const Ray &r, int k, int kfirst, int kend, int kwalk0,
                                        float s_start, double &s, double &s1) {
  const int w = __ldg(&a.trav[k].x);
  s = k == kwalk0 ? (double)s_start : cell_event64(r, __ldg(&a.trav[k - 1].x), w);
  if (k == kwalk0 && k > kfirst && s_start == __int_as_float(__ldg(&a.trav[k - 1].y)))
    s = cell_event64(r, __ldg(&a.trav[k - 1].x), w);   // (the walk started on the boundary itself)
  s1 = k + 1 < kend ? cell_event64(r, w, __ldg(&a.trav[k + 1].x)) : exit64(r, a.tc.nx, a.tc.ny, a.tc.z_top);
}

// Crossing records of one chain x ray: up to RCAP per surface, kept in shared
// memory at slot [(l*RCAP + m)*MT_THREADS + tid] (conflict-free: consecutive
// threads, consecutive 16-B words).
#ifndef MT_RCAP
#define MT_RCAP 3
#endif
#ifndef MT_RL_GLOBAL_H
#define MT_RL_GLOBAL_H 1
#endif
#ifndef MT_RL_MINB
#define MT_RL_MINB 4
#endif
#ifndef RL_KM
#define RL_KM 1   // ray lanes use solve32k (K, M from the cell geometry; -1.8% vs solve32)
#endif
// lanes per deferred pair in k_trace_defer: 8 after the chain lanes (many pairs,
// throughput), more after the ray lanes (few pairs, latency of the band rounds)
#ifndef DEFER_DG
#define DEFER_DG 8
#endif
#ifndef DEFER_DG_RL
#define DEFER_DG_RL 16
#endif
#ifndef DEFER_SMALL_R
#define DEFER_SMALL_R 65536   // at most this many rays: 32 lanes per deferred pair
#endif
#ifndef MT_CL_MINB
#define MT_CL_MINB 5
#endif
#ifndef V0_SOLVE
#define V0_SOLVE 1
#endif
#ifndef V0_LAUNDER
#define V0_LAUNDER 1
#endif
#ifndef V0_TILE
#define V0_TILE 0
#endif
constexpr int RCAP = MT_RCAP;

// G_l[node] += w φ_node(u, v) for the cell's 4 corners (a6), fixed point:
// w is prescaled by MT_GQ (R30).
__device__ __forceinline__ void scatter4(macc *Gl, int STRIDE, int base, int ny, float w, float u, float v) {
  const float wa = w * (1.f - u), wb = w * u;
  atomicAdd(Gl + base * STRIDE, q_raw(wa * (1.f - v)));
  atomicAdd(Gl + (base + ny) * STRIDE, q_raw(wb * (1.f - v)));
  atomicAdd(Gl + (base + 1) * STRIDE, q_raw(wa * v));
  atomicAdd(Gl + (base + ny + 1) * STRIDE, q_raw(wb * v));
}

// ---------------------------------------------------------------------------
// generic walk (ray lanes, deferred pairs): one chain x ray, thread-serial.
// Heights of the chain at Hk with node stride STRIDE (1: a shared-memory tile,
// 32: the chain-interleaved global layout).  Ill-conditioned cells are
// re-solved in place in fp64.  SCAT: scatter f_l φ/|g'| directly into Gk;
// else record crossings (n[l] counts all, the first RCAP are stored).
// ---------------------------------------------------------------------------
template <int STRIDE, bool SCAT>
__device__ __forceinline__ void walk(const TraceArgs *ta, int kfirst, const Ray &r, const int2 *__restrict__ cells,
                                     const float4 *__restrict__ cgeo, int k, int kend, float s0,
                                     float s_in0, float s_hi, int ny, int N, const float *Hk,
                                     const float *Hlo, macc *Gk, float4 bd, float &B0, float &B1,
                                     float4 *rec, int *n, float f0, float f1) {
  float s = s0, ds = s0 - s_in0;
  const int kwalk0 = k;
  for (; k < kend; k++) {
    const int2 w = __ldg(cells + k);
    const float s1 = __int_as_float(w.y);
    const float4 cg = shift_geo(__ldg(cgeo + k), ds);
    const int i = cell_i(w.x), j = cell_j(w.x), base = i * ny + j;
    const float za = s * r.dz, zb = s1 * r.dz, Ls = s1 - s;
#pragma unroll
    for (int l = 0; l < 2; l++) {
      const float zmin = l ? bd.z : bd.x, zmax = l ? bd.w : bd.y;
      float &B = l ? B1 : B0;
      if (zb <= zmin) { B += Ls; continue; }
      if (za >= zmax) continue;
      const float *p = Hk + (size_t)l * N * STRIDE + base * STRIDE;
      const float h00 = p[0], h10 = p[ny * STRIDE], h01 = p[STRIDE], h11 = p[ny * STRIDE + STRIDE];
      if (zb <= fminf(fminf(h00, h10), fminf(h01, h11))) { B += Ls; continue; }
      if (za >= fmaxf(fmaxf(h00, h10), fmaxf(h01, h11))) continue;
      macc *Gl = SCAT ? Gk + (size_t)l * N * STRIDE : nullptr;
      const float f = l ? f1 : f0;
      auto emit = [&](float u, float v, float ig) {
        if (SCAT) {
          scatter4(Gl, STRIDE, base, ny, f * ig, u, v);
        } else {
          if (n[l] < RCAP) rec[(l * RCAP + n[l]) * MT_THREADS] = make_float4(__int_as_float(base), u, v, ig);
          n[l]++;
        }
      };
      if (!solve32(h00, h10, h01, h11, cg, za, Ls, r.dz, B, emit)) {
        // fp64 heights = fp32 value + stored residual (chain-interleaved column, stride 32)
        const float *pl = Hlo + ((size_t)l * N + base) * 32;
        double se, se1;
        piece64(*ta, r, k, kfirst, kend, kwalk0, s0, se, se1);
        const Fix x = fix64((double)h00 + pl[0], (double)h10 + pl[ny * 32], (double)h01 + pl[32],
                            (double)h11 + pl[ny * 32 + 32], sgeo[0][i], sgeo[0][i + 1], sgeo[1][j],
                            sgeo[1][j + 1], r, se, se1);
        B += x.below;
        for (int m = 0; m < x.n; m++) emit(x.u[m], x.v[m], x.ig[m]);
      }
    }
    if (s1 >= s_hi) break;
    s = s1;
    ds = 0.f;
  }
}

// First stored cell of the ray whose s_out exceeds s (binary search; the last
// cell's s_out is s_exit > s), and the entry s_in of that cell.
__device__ __forceinline__ int band_entry(const int2 *__restrict__ cells, int lo, int hi, float s,
                                          float &s_in) {
  const int first = lo;
  hi -= 1;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (__int_as_float(__ldg(&cells[mid].y)) > s) hi = mid;
    else lo = mid + 1;
  }
  s_in = lo > first ? __int_as_float(__ldg(&cells[lo - 1].y)) : 0.f;
  return lo;
}

// Queue overflow: mark pair (c, ray) in the (C x R)-bit redo bitmap.
__device__ __forceinline__ void redo_mark(const TraceArgs &a, int c, int rr) {
  const int64_t idx = (int64_t)c * a.R + rr;
  atomicOr(a.redo + (idx >> 5), 1u << (idx & 31));
}

// Fused epilogue (a4-a5): t = ln(λ/C) (C > 0) or ln λ (C = 0) from the
// per-ray constant t_base (HP4, R15); returns ℓ_p, sets ∂ℓ/∂O = (λ - C)/Λ.
__device__ __forceinline__ float epilogue(float tb, float cnt, const TraceConsts &tc, float B0,
                                          float B1, float &dldO) {
  const float t = tb - (tc.k0 * B0 + tc.k1 * B1) * tc.inv_att;
  if (cnt > 0.f) {
    // ℓ = -C (e^t - 1 - t); e^t - 1 - t by its series when |t| < 0.1 (truncation
    // < 2e-10 relative), expm1f otherwise
    float d;
    if (fabsf(t) < 0.1f)
      d = t * t * fmaf(t, fmaf(t, fmaf(t, fmaf(t, 1.f / 720.f, 1.f / 120.f), 1.f / 24.f), 1.f / 6.f), 0.5f);
    else
      d = expm1f(t) - t;
    dldO = cnt * (d + t) * tc.inv_att;
    return -cnt * d;
  }
  const float lam = __expf(t);
  dldO = lam * tc.inv_att;
  return -lam;
}

__device__ __forceinline__ void load_geometry(const TraceArgs &a) {   // -> sgeo (indexed directly)
  const int nx = a.tc.nx, ny = a.tc.ny;
  for (int k = threadIdx.x; k < nx; k += blockDim.x) {
    sgeo[0][k] = a.X[k];
    sgeo[2][k] = k < nx - 1 ? 1.f / (a.X[k + 1] - a.X[k]) : 0.f;
  }
  for (int k = threadIdx.x; k < ny; k += blockDim.x) {
    sgeo[1][k] = a.Y[k];
    sgeo[3][k] = k < ny - 1 ? 1.f / (a.Y[k + 1] - a.Y[k]) : 0.f;
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// traversal builder (create time): thread = ray; count pass then write pass
// ---------------------------------------------------------------------------
__global__ void k_build_trav(TraceArgs a, const int32_t *off, int32_t *count, int2 *cells, float4 *cgeo,
                             float2 *ckm,
                             int2 *rl_head, uint4 *rl_code, uint32_t *rl_ovf,
                             const int32_t *ovf_off) {
  __shared__ float Xs[MT_MAX_AXIS], Ys[MT_MAX_AXIS];
  const int nx = a.tc.nx, ny = a.tc.ny;
  for (int k = threadIdx.x; k < nx; k += blockDim.x) Xs[k] = a.X[k];
  for (int k = threadIdx.x; k < ny; k += blockDim.x) Ys[k] = a.Y[k];
  __syncthreads();
  int64_t rr = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (rr >= a.R) return;
  DdaRay q = dda_ray(load_ray(a.ray_a, a.ray_b, rr));
  int i = start_axis(Xs, nx, q.r.ox, q.r.dx), j = start_axis(Ys, ny, q.r.oy, q.r.dy);
  float s = 0.f, s_in = 0.f;   // s_in: the previous STORED s_out (what the walks carry)
  int n = 0;
  if (rl_head) rl_head[rr] = make_int2((off[rr + 1] - off[rr]) | (i << 8) | (j << 15), ovf_off[rr]);
  uint32_t cw[4] = {0u, 0u, 0u, 0u};
  for (int guard = 0; guard < 4 * (MT_MAX_AXIS + 2); guard++) {
    float s_ev;
    int fc;
    int ev = dda_next(q, i, j, Xs, Ys, nx, ny, a.tc.z_top, s_ev, &fc);
    if (rl_code) {   // 2-bit exit code of cell n: 0 top (s_exit), 1 x-line, 2 y-line, 3 vertex
      if (n < 64) cw[n >> 4] |= (uint32_t)fc << (2 * (n & 15));
      else atomicOr(rl_ovf + ovf_off[rr] + ((n - 64) >> 4), (uint32_t)fc << (2 * (n & 15)));
    }
    float s1 = fminf(s_ev, q.r.s_exit);
    const float so = fmaxf(s1, s);
    if (cells) {
      // cell-local entry point and rates (a0), fp64 from the exact fp32 inputs, and the
      // ray-only parts of the cell solve's g1 and g2 (K = u β + v α, M = α β)
      const double ix = 1.0 / ((double)Xs[i + 1] - (double)Xs[i]);
      const double iy = 1.0 / ((double)Ys[j + 1] - (double)Ys[j]);
      const double u = ((double)q.r.ox + (double)s_in * (double)q.r.dx - (double)Xs[i]) * ix;
      const double v = ((double)q.r.oy + (double)s_in * (double)q.r.dy - (double)Ys[j]) * iy;
      const float uf = (float)u, vf = (float)v, af = (float)((double)q.r.dx * ix), bf = (float)((double)q.r.dy * iy);
      cells[off[rr] + n] = make_int2(cell_pack(i, j, ny), __float_as_int(so));
      cgeo[off[rr] + n] = make_float4(uf, vf, af, bf);
      ckm[off[rr] + n] = make_float2((float)((double)uf * bf + (double)vf * af), (float)((double)af * bf));
    }
    s_in = so;
    n++;
    if (ev & 4) break;
    if (ev & 1) i += q.sx;
    if (ev & 2) j += q.sy;
    s = s1;
  }
  if (count) count[rr] = n;
  if (rl_code) rl_code[rr] = make_uint4(cw[0], cw[1], cw[2], cw[3]);
}

// ---------------------------------------------------------------------------
// K2, chain lanes: warp = one ray x 32 (k_trace_v0) or 64 (k_trace_c2) chains
// ---------------------------------------------------------------------------
// Per evaluation, k_cell_prep writes the paired heights the chain-lanes walk
// reads: H2 = (H_l(i,j), H_l(i,j+1)) per node, [group][l][node][lane], so a
// cell's four corners of one surface are two 8-B loads of one 256-B line each.
__global__ void __launch_bounds__(MT_THREADS) k_cell_prep(const float *__restrict__ H, float2 *__restrict__ H2, int ny,
                                                        int64_t n) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // [group][l][node][lane]
  if (t >= n) return;
  const int node_j = (int)((t >> 5) % ny);
  H2[t] = make_float2(H[t], node_j + 1 < ny ? H[t + 32] : 0.f);
}

template <bool FAST>
__device__ __forceinline__ void scatter_recs(const float4 *rec, int m0, int m1, macc *G0, int N, int oy, float f0,
                                             float f1) {
#pragma unroll 1
  for (int m = 0; m < m0 + m1; m++) {
    const int l = m >= m0;
    const float4 q = rec[(l ? RCAP + m - m0 : m) * MT_THREADS];
    const float wv = (l ? f1 : f0) * q.w, u = q.y, v = q.z, wa = wv * (1.f - u), wb = wv * u;
    macc *pg = G0 + (l ? N * 32 : 0) + (__float_as_uint(q.x) << 5);
    if (FAST) {
      atomicAdd(pg, q_small(wa * (1.f - v)));
      atomicAdd(pg + oy, q_small(wb * (1.f - v)));
      atomicAdd(pg + 32, q_small(wa * v));
      atomicAdd(pg + oy + 32, q_small(wb * v));
    } else {
      atomicAdd(pg, q_raw(wa * (1.f - v)));
      atomicAdd(pg + oy, q_raw(wb * (1.f - v)));
      atomicAdd(pg + 32, q_raw(wa * v));
      atomicAdd(pg + oy + 32, q_raw(wb * v));
    }
  }
}

// ---- round-1 chain-lanes kernel (A/B baseline while the new one is tuned) ----
// Same, warp-cooperative (chain lanes, all 32 lanes converged, uniform
// arguments): one coalesced load of 32 cells and a ballot per round.
__device__ __forceinline__ int band_entry_warp(const int2 *__restrict__ cells, int lo, int hi, float s,
                                               float &s_in) {
  const int lane = threadIdx.x & 31;
  float prev = 0.f;   // s_out of the cell before this round (0 before the first cell)
  for (int b = lo; b < hi; b += 32) {
    const int k = b + lane;
    const float so = k < hi ? __int_as_float(__ldg(&cells[k].y)) : 3.0e38f;
    const unsigned m = __ballot_sync(0xffffffffu, so > s);
    const float before = __shfl_up_sync(0xffffffffu, so, 1);
    if (m) {
      const int f = __ffs(m) - 1;
      const float sb = __shfl_sync(0xffffffffu, before, f);
      s_in = f > 0 ? sb : prev;
      return b + f;
    }
    prev = __shfl_sync(0xffffffffu, so, 31);
  }
  s_in = prev;
  return hi - 1;
}

// ---------------------------------------------------------------------------
// One surface of one stored cell for this lane's chain.  Warp-uniform inputs:
// the cell word w (node offset, i, j), its geometry cg, the piece [s, s1] of
// the ray (za = s d_z, zb = s1 d_z).  Per lane: the chain's heights (column of
// the chain-interleaved layout), its band [zmin, zmax] of this surface, B.  An
// ill-conditioned cell sets `defer`: the whole chain x ray pair is then handed
// to k_trace_defer (same fp32 cell code plus in-place fp64 re-solves), so the
// hot kernel holds no double-precision code and makes no calls (a call forces
// the ABI's spills into the loop).
template <int L, bool KM = false>
__device__ __forceinline__ void cw_solve(float4 h, int w, float4 cg, float za, float zb, float Ls,
                                         float dz, float &B, int &n, int &defer, float4 *rec,
                                         float2 km = make_float2(0.f, 0.f)) {
  const float h00 = h.x, h01 = h.y, h10 = h.z, h11 = h.w;
  if (zb <= fminf(fminf(h00, h10), fminf(h01, h11))) { B += Ls; return; }   // bilinear min at a corner
  if (za >= fmaxf(fmaxf(h00, h10), fmaxf(h01, h11))) return;
  const float wbase = __int_as_float(cell_off32(w) >> 5);
  auto emit = [&](float u, float v, float ig) {
    if (n < RCAP) rec[(L * RCAP + n) * MT_THREADS] = make_float4(wbase, u, v, ig);
    n++;
  };
  if (KM) {
    if (!solve32k(h00, h10, h01, h11, cg, km, za, Ls, dz, B, emit)) defer = 1;
  } else if (!solve32(h00, h10, h01, h11, cg, za, Ls, dz, B, emit)) {
    defer = 1;
  }
}

// Second pass of a pair with more than RCAP crossings of a surface (dℓ/dO now
// known): the same cell code, crossings m >= RCAP scattered directly (the
// first RCAP were stored and scattered from the records).
__device__ __forceinline__ void cw_scatter_surface(const float *__restrict__ Hg, unsigned off, int oy, float4 cg,
                                                   float za, float zb, float Ls, float dz, float zmin, float zmax,
                                                   macc *Gp, float f, int &m, float2 km) {
  if (zb <= zmin || za >= zmax) return;
  const float *p = Hg + off;
  const float h00 = __ldg(p), h01 = __ldg(p + 32), h10 = __ldg(p + oy), h11 = __ldg(p + oy + 32);
  if (zb <= fminf(fminf(h00, h10), fminf(h01, h11))) return;
  if (za >= fmaxf(fmaxf(h00, h10), fmaxf(h01, h11))) return;
  float Bd = 0.f;
  auto emit = [&](float u, float v, float ig) {
    if (m >= RCAP) {
      const float wv = f * ig, wa = wv * (1.f - u), wb = wv * u;
      atomicAdd(Gp, q_raw(wa * (1.f - v)));
      atomicAdd(Gp + oy, q_raw(wb * (1.f - v)));
      atomicAdd(Gp + 32, q_raw(wa * v));
      atomicAdd(Gp + oy + 32, q_raw(wb * v));
    }
    m++;
  };
  // the same solve as the first walk (V0_SOLVE), so crossing m is the same crossing
  if (V0_SOLVE) solve32k(h00, h10, h01, h11, cg, km, za, Ls, dz, Bd, emit);
  else solve32(h00, h10, h01, h11, cg, za, Ls, dz, Bd, emit);
}

template <int L>
__device__ __forceinline__ void cw_surface(const float *__restrict__ Hg, unsigned off, int w, int oy,
                                           float4 cg, float za, float zb, float Ls, float dz, float zmin,
                                           float zmax, float &B, int &n, int &defer, float4 *rec, float2 km) {
  if (zb <= zmin) { B += Ls; return; }            // below the chain's lowest node of this surface
  if (za >= zmax) return;                         // above its highest node
  // paired heights: element k holds (H(i,j), H(i,j+1)), so a cell's four corners are two 8-byte loads.
  // Hg is the chain group's (warp-uniform) base and off the cell's uniform offset + the lane.
  const float2 *p2 = reinterpret_cast<const float2 *>(Hg) + off;
  const float2 r0 = __ldg(p2), r1 = __ldg(p2 + oy);
  cw_solve<L, V0_SOLVE>(make_float4(r0.x, r0.y, r1.x, r1.y), w, cg, za, zb, Ls, dz, B, n, defer, rec, km);
}


template <int MODE, int NY>
__global__ void __launch_bounds__(MT_THREADS, MT_CL_MINB) k_trace_v0(TraceArgs a) {
  extern __shared__ __align__(16) float4 recs[];    // crossing records [2*RCAP][MT_THREADS]
  const int ny = NY ? NY : a.tc.ny, N = a.tc.N;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#if V0_TILE
  // block order: tiles of V0_TILE ray chunks x all chain groups (L2 reuse of the chunk's
  // traversal records across groups)
  const int lin = blockIdx.y * gridDim.x + blockIdx.x, G_ = gridDim.y;
  const int tile = lin / (G_ * V0_TILE), within = lin - tile * (G_ * V0_TILE);
  const int grp = within / V0_TILE, chunk = tile * V0_TILE + (within - (within / V0_TILE) * V0_TILE);
#else
  const int grp = blockIdx.y, chunk = blockIdx.x;
#endif
  const int c = grp * 32 + lane;
  const bool act = c < a.C;
  float4 *rec = recs + threadIdx.x;

  // this lane's chain band; the warp walks the union band of its 32 chains.
  // Inactive lanes get a band that every cell lies "above" (no loads).
  float4 bd = act ? __ldg(a.band + c) : make_float4(3.0e38f, -3.0e38f, 3.0e38f, -3.0e38f);
  float zlo = bd.x, zhi = bd.w;
  for (int o = 16; o > 0; o >>= 1) {
    zlo = fminf(zlo, __shfl_xor_sync(0xffffffffu, zlo, o));
    zhi = fmaxf(zhi, __shfl_xor_sync(0xffffffffu, zhi, o));
  }
  if (!act) bd = make_float4(-3.0e38f, -3.0e38f, -3.0e38f, -3.0e38f);
  const int oy = ny * 32;
  const unsigned gbase = (unsigned)grp * 2 * N * 32 + lane;   // this lane's column of the group tile
  const float2 *__restrict__ H2g = reinterpret_cast<const float2 *>(a.cl) + (size_t)grp * 2 * N * 32;
#if V0_LAUNDER
  // opaque copy: otherwise the compiler rematerialises this base from CTAID and the kernel
  // parameters at every corner load (12 uniform-datapath instructions per surface-cell)
  asm volatile("mov.b64 %0, %0;" : "+l"(H2g));
#endif
  const float2 *__restrict__ H2g1 = H2g + (size_t)N * 32;   // warp-uniform bases of the two surfaces
  macc llq = 0;

  const int r_begin = chunk * (int)a.rays_per_block;
  const int r_end = min((int)a.R, r_begin + (int)a.rays_per_block);
  for (int rr = r_begin + warp; rr < r_end; rr += MT_THREADS / 32) {
    float dz, s_exit;
    {
      const float2 rb = __ldg(reinterpret_cast<const float2 *>(a.ray_b + rr));   // broadcast
      dz = rb.x; s_exit = rb.y;
    }
    // band bounds, widened by 1e-6 so fast division can only walk more cells
    const float s_lo = fminf(__fdividef(zlo, dz) * (1.f - 1e-6f), s_exit);
    const float s_hi = fminf(__fdividef(zhi, dz) * (1.f + 1e-6f), s_exit);
    float B0 = s_lo, B1 = s_lo;                        // below both surfaces before s_lo
    int n0 = 0, n1 = 0, defer = 0;
    if (s_lo < s_exit) {                               // warp-uniform
      const int kend = __ldg(a.trav_off + rr + 1);
      float s_in0;
      const int k0 = band_entry_warp(a.trav, __ldg(a.trav_off + rr), kend, s_lo, s_in0);
      float s = s_lo, za = s_lo * dz, ds = s_lo - s_in0;
      for (int k = k0; k < kend; k++) {
        // (a zero-length stored cell, possible only through fp32 event rounding
        // in the builder, adds nothing: no crossing, B += 0)
        const int2 w = __ldg(a.trav + k);
        const float4 cg = shift_geo(__ldg(a.trav_geo + k), ds);
        const float s1 = __int_as_float(w.y);
        const float zb = s1 * dz, Ls = s1 - s;
        float2 km = make_float2(0.f, 0.f);
        if (V0_SOLVE) {
          km = __ldg(a.trav_km + k);
          km.x = fmaf(2.f * km.y, ds, km.x);   // K of the shifted entry point (first cell only)
        }
        // uniform group base (a scalar register pair) + the cell's offset + the lane
        const unsigned offl = cell_off32(w.x) + (unsigned)lane;
        cw_surface<0>(reinterpret_cast<const float *>(H2g), offl, w.x, oy, cg, za, zb, Ls, dz, bd.x, bd.y, B0, n0,
                      defer, rec, km);
        cw_surface<1>(reinterpret_cast<const float *>(H2g1), offl, w.x, oy, cg, za, zb, Ls, dz, bd.z, bd.w, B1, n1,
                      defer, rec, km);

        if (s1 >= s_hi) break;
        s = s1;
        za = zb;
        ds = 0.f;
      }
    }
    // an ill-conditioned cell: the whole pair goes to k_trace_defer (fp64 re-solve)
    if (defer) {
      const int q = atomicAdd(a.ovf_n, 1);
      if (q < a.ovf_cap) a.ovf_q[q] = make_float4(__int_as_float(c), __int_as_float(rr), s_lo, s_hi);
      else redo_mark(a, c, rr);   // queue full: the follow-up kernel finds the pair in the bitmap
    }
    if (MODE == TRACE_LL) {
      const bool over = !defer && (n0 > RCAP || n1 > RCAP);   // more crossings than records
      float f0 = 0.f, f1 = 0.f;
      macc *G0 = a.G + (size_t)grp * 2 * N * 32 + lane;
      if (!defer && act) {
        const float2 rb = __ldg(reinterpret_cast<const float2 *>(a.ray_b + rr) + 1);
        float dldO;
        llq += q_ll(epilogue(rb.x, rb.y, a.tc, B0, B1, dldO));
        f0 = dldO * a.tc.k0 * (float)MT_GQ;
        f1 = dldO * a.tc.k1 * (float)MT_GQ;
        for (int m = 0; m < min(n0, RCAP); m++) {
          const float4 q = rec[m * MT_THREADS];
          const float w = f0 * q.w, u = q.y, v = q.z;
          macc *pg = G0 + ((unsigned)__float_as_int(q.x) << 5);
          const float wa = w * (1.f - u), wb = w * u;
          atomicAdd(pg, q_raw(wa * (1.f - v)));
          atomicAdd(pg + oy, q_raw(wb * (1.f - v)));
          atomicAdd(pg + 32, q_raw(wa * v));
          atomicAdd(pg + oy + 32, q_raw(wb * v));
        }
        macc *G1 = G0 + N * 32;
        for (int m = 0; m < min(n1, RCAP); m++) {
          const float4 q = rec[(RCAP + m) * MT_THREADS];
          const float w = f1 * q.w, u = q.y, v = q.z;
          macc *pg = G1 + ((unsigned)__float_as_int(q.x) << 5);
          const float wa = w * (1.f - u), wb = w * u;
          atomicAdd(pg, q_raw(wa * (1.f - v)));
          atomicAdd(pg + oy, q_raw(wb * (1.f - v)));
          atomicAdd(pg + 32, q_raw(wa * v));
          atomicAdd(pg + oy + 32, q_raw(wb * v));
        }
      }
      if (__any_sync(0xffffffffu, over)) {   // wide bands (e.g. prior draws): re-walk, scatter the rest
        const int kend = __ldg(a.trav_off + rr + 1);
        float s_in0;
        const int k0 = band_entry_warp(a.trav, __ldg(a.trav_off + rr), kend, s_lo, s_in0);
        float s = s_lo, za = s_lo * dz, ds = s_lo - s_in0;
        int m0 = 0, m1 = 0;
        for (int k = k0; k < kend; k++) {
          const int2 w = __ldg(a.trav + k);
          const float4 cg = shift_geo(__ldg(a.trav_geo + k), ds);
          const float s1 = __int_as_float(w.y);
          const float zb = s1 * dz, Ls = s1 - s;
          if (over) {
            float2 km = __ldg(a.trav_km + k);
            km.x = fmaf(2.f * km.y, ds, km.x);
            const unsigned off = cell_off32(w.x) + gbase;
            macc *pg = G0 + ((unsigned)(cell_off32(w.x)));
            if (n0 > RCAP) cw_scatter_surface(a.H, off, oy, cg, za, zb, Ls, dz, bd.x, bd.y, pg, f0, m0, km);
            if (n1 > RCAP) cw_scatter_surface(a.H, off + N * 32, oy, cg, za, zb, Ls, dz, bd.z, bd.w,
                                              pg + N * 32, f1, m1, km);
          }
          if (s1 >= s_hi) break;
          s = s1;
          za = zb;
          ds = 0.f;
        }
      }
    } else if (act && !defer) {
      const int64_t o = (int64_t)c * a.R + __ldg(a.perm + rr);
      a.Lout[3 * o + 0] = B0;
      a.Lout[3 * o + 1] = B1 - B0;
      a.Lout[3 * o + 2] = s_exit - B1;
      a.Oout[o] = a.tc.k0 * B0 + a.tc.k1 * B1 + a.obase[rr];
    }
  }
  if (MODE == TRACE_LL && act) atomicAdd(a.ll + c, llq);
}

// ---------------------------------------------------------------------------
// K2, chain lanes with two chains per lane (C >= 64): warp = one ray x 64
// chains, lane l = chains 64g + l and 64g + 32 + l.  The ray's traversal,
// band entry, cell records and loop control are shared by twice as many
// chains as in k_trace_v0, and each lane carries two independent solve
// chains (latency hiding).  Paired heights of both chains in one 16-B load:
// [g64][l][node][lane] float4 {H_A(i,j), H_A(i,j+1), H_B(i,j), H_B(i,j+1)}
// (k_cell_prep2).  Blocks run in tiles of C2_TILE ray chunks x all chain
// groups, so a chunk's traversal records are reused from L2 by every group.
// ---------------------------------------------------------------------------
#ifndef C2_TILE
#define C2_TILE 1
#endif
#ifndef C2_RCAP
#define C2_RCAP 1   // crossing records per (chain, surface); more re-walk in-kernel (see launch_c2)
#endif
#ifndef C2_KMC
#define C2_KMC 1   // K, M of solve32k formed in-lane from the cell geometry: no trav_km load (-0.9%)
#endif
#ifndef C2_THREADS
#define C2_THREADS 256   // threads per block of k_trace_c2
#endif
#ifndef C2_MINB
#define C2_MINB (1024 / C2_THREADS)
#endif


__global__ void __launch_bounds__(MT_THREADS) k_cell_prep2(const float *__restrict__ H, float4 *__restrict__ H4, int C,
                                                         int ny, int N, int64_t n) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // [g64][l][node][lane]
  if (t >= n) return;
  const int lane = (int)(t & 31);
  const int64_t q = t >> 5;
  const int node = (int)(q % N), l = (int)((q / N) & 1), g = (int)(q / (2 * (int64_t)N));
  const int j = node % ny;
  float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int v = 0; v < 2; v++) {
    const int c = g * 64 + v * 32 + lane;
    if (c < C) {
      const float *p = H + (((size_t)(c >> 5) * 2 + l) * N + node) * 32 + lane;
      const float h0 = p[0], h1 = j + 1 < ny ? p[32] : 0.f;
      if (v == 0) { o.x = h0; o.y = h1; } else { o.z = h0; o.w = h1; }
    } else if (v == 0) {
      o.x = o.y = -3.0e38f;   // never loaded: the lane-union band skips inactive chains
    } else {
      o.z = o.w = -3.0e38f;
    }
  }
  H4[t] = o;
}

// One chain's surface-cell from its corners (the corner-bound test, then the solve).
template <int SLOT, bool SCAT>
__device__ __forceinline__ void c2_cell(float h00, float h01, float h10, float h11, float4 cg, float2 km, float za,
                                        float zb, float Ls, float dz, float wbase, float &B, int &n, int &defer,
                                        float4 *rec, macc *Gp, int oy, float f) {
  if (zb <= fminf(fminf(h00, h10), fminf(h01, h11))) { B += Ls; return; }   // bilinear min at a corner
  if (za >= fmaxf(fmaxf(h00, h10), fmaxf(h01, h11))) return;
  auto emit = [&](float u, float v, float ig) {
    if (SCAT) {
      if (n >= C2_RCAP) {
        const float wv = f * ig, wa = wv * (1.f - u), wb = wv * u;
        atomicAdd(Gp, q_raw(wa * (1.f - v)));
        atomicAdd(Gp + oy, q_raw(wb * (1.f - v)));
        atomicAdd(Gp + 32, q_raw(wa * v));
        atomicAdd(Gp + oy + 32, q_raw(wb * v));
      }
    } else if (n < C2_RCAP) {
      rec[(SLOT * C2_RCAP + n) * C2_THREADS] = make_float4(wbase, u, v, ig);
    }
    n++;
  };
  if (!solve32k(h00, h10, h01, h11, cg, km, za, Ls, dz, B, emit)) defer = 1;
}

// Crossing records of k_trace_c2, [chain v][surface l][C2_RCAP][thread] (static:
// the slot address is a constant offset from the thread's, no shared-window
// pointer to rematerialise).
__shared__ __align__(16) float4 c2_recs[4 * C2_RCAP][C2_THREADS];

// Same, with the lane's crossing counters and defer flags packed in one register
// (fields of 5 bits, saturating at 31: n0A @0, n1A @5, n0B @10, n1B @15; defer
// bits 20 / 21); records of (chain v, surface l) at slots slot0 = (2v + l) RCAP.
__device__ __forceinline__ void c2_cellp(float h00, float h01, float h10, float h11, float4 cg, float2 km, float za,
                                         float zb, float Ls, float dz, float wbase, float &B, unsigned &cnt,
                                         const int sh, const unsigned dbit, const int slot0) {
  if (zb <= fminf(fminf(h00, h10), fminf(h01, h11))) { B += Ls; return; }   // bilinear min at a corner
  if (za >= fmaxf(fmaxf(h00, h10), fmaxf(h01, h11))) return;
  auto emit = [&](float u, float v, float ig) {
    const unsigned n = (cnt >> sh) & 31u;
    if (n < C2_RCAP) c2_recs[slot0 + n][threadIdx.x] = make_float4(wbase, u, v, ig);
    if (n < 31u) cnt += 1u << sh;
  };
  if (!solve32k(h00, h10, h01, h11, cg, km, za, Ls, dz, B, emit)) cnt |= dbit;
}

// The ray loop of k_trace_c2; FULL: both chains of every lane are active (every
// 64-chain group but a ragged last one), so the per-chain guards compile away.
template <int MODE, bool FULL>
__device__ __forceinline__ void c2_rays(const TraceArgs &a, int N, int oy, const int g, const int chunk,
                                        const int acts, const float4 bd, const float zlo, const float zhi,
                                        const float4 *__restrict__ H4, float &sllA, float &sllB) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cA = g * 64 + lane, cB = cA + 32;
  const bool actA = FULL || (acts & 1), actB = FULL || (acts & 2);
  const int r_begin = chunk * (int)a.rays_per_block;
  const int r_end = min((int)a.R, r_begin + (int)a.rays_per_block);
  for (int rr = r_begin + warp; rr < r_end; rr += C2_THREADS / 32) {
    const float2 rb0 = __ldg(reinterpret_cast<const float2 *>(a.ray_b + rr));
    const float dz = rb0.x, s_exit = rb0.y;
    const float s_lo = fminf(__fdividef(zlo, dz) * (1.f - 1e-6f), s_exit);
    const float s_hi = fminf(__fdividef(zhi, dz) * (1.f + 1e-6f), s_exit);
    float B0A = s_lo, B1A = s_lo, B0B = s_lo, B1B = s_lo;
    unsigned cnt = 0;   // packed counters / defer flags (c2_cellp)
    if (s_lo < s_exit) {
      const int kend = __ldg(a.trav_off + rr + 1), kbeg = __ldg(a.trav_off + rr);
      float s_in0;
      const int k0 = band_entry_warp(a.trav, kbeg, kend, s_lo, s_in0);
      float s = s_lo, za = s_lo * dz, ds = s_lo - s_in0;
      for (int k = k0; k < kend; k++) {
        const int2 w = __ldg(a.trav + k);
        const float4 cg = shift_geo(__ldg(a.trav_geo + k), ds);
        float2 km = C2_KMC ? make_float2(fmaf(cg.x, cg.w, cg.y * cg.z), cg.z * cg.w) : __ldg(a.trav_km + k);
        if (!C2_KMC) km.x = fmaf(2.f * km.y, ds, km.x);
        const float s1 = __int_as_float(w.y);
        const float zb = s1 * dz, Ls = s1 - s;
        const unsigned off = cell_off32(w.x);
        const float wb = __uint_as_float(off >> 5);
#pragma unroll
        for (int l = 0; l < 2; l++) {
          const float zmin = l ? bd.z : bd.x, zmax = l ? bd.w : bd.y;
          float &BA = l ? B1A : B0A, &BB = l ? B1B : B0B;
          if (zb <= zmin) { BA += Ls; BB += Ls; continue; }   // below both chains' lowest node
          if (za >= zmax) continue;                            // above both chains' highest node
          const float4 *p = H4 + (size_t)l * N * 32 + off;
          const float4 r0 = __ldg(p), r1 = __ldg(p + oy);
          if (actA) c2_cellp(r0.x, r0.y, r1.x, r1.y, cg, km, za, zb, Ls, dz, wb, BA, cnt, l ? 5 : 0, 1u << 20,
                             l * C2_RCAP);
          if (actB) c2_cellp(r0.z, r0.w, r1.z, r1.w, cg, km, za, zb, Ls, dz, wb, BB, cnt, l ? 15 : 10, 1u << 21,
                             (2 + l) * C2_RCAP);
        }
        if (s1 >= s_hi) break;
        s = s1;
        za = zb;
        ds = 0.f;
      }
    }
    const int dA = (cnt >> 20) & 1, dB = (cnt >> 21) & 1;
    const int n0A = cnt & 31, n1A = (cnt >> 5) & 31, n0B = (cnt >> 10) & 31, n1B = (cnt >> 15) & 31;
    if (dA) {
      const int q = atomicAdd(a.ovf_n, 1);
      if (q < a.ovf_cap) a.ovf_q[q] = make_float4(__int_as_float(cA), __int_as_float(rr), s_lo, s_hi);
      else redo_mark(a, cA, rr);
    }
    if (dB) {
      const int q = atomicAdd(a.ovf_n, 1);
      if (q < a.ovf_cap) a.ovf_q[q] = make_float4(__int_as_float(cB), __int_as_float(rr), s_lo, s_hi);
      else redo_mark(a, cB, rr);
    }
    if (MODE == TRACE_LL) {
      const bool overA = !dA && (n0A > C2_RCAP || n1A > C2_RCAP), overB = !dB && (n0B > C2_RCAP || n1B > C2_RCAP);
      float f0A = 0.f, f1A = 0.f, f0B = 0.f, f1B = 0.f;
      macc *GA = a.G + (size_t)(2 * g) * 2 * N * 32 + lane, *GB = GA + (size_t)2 * N * 32;
      const float2 rt = __ldg(reinterpret_cast<const float2 *>(a.ray_b + rr) + 1);
#pragma unroll
      for (int v = 0; v < 2; v++) {
        if (v ? (dB || !actB) : (dA || !actA)) continue;
        float dldO;
        const float ll = epilogue(rt.x, rt.y, a.tc, v ? B0B : B0A, v ? B1B : B1A, dldO);
        const float f0 = dldO * a.tc.k0 * (float)MT_GQ, f1 = dldO * a.tc.k1 * (float)MT_GQ;
        if (v) sllB += ll; else sllA += ll;
        if (v) { f0B = f0; f1B = f1; } else { f0A = f0; f1A = f1; }
#pragma unroll
        for (int l = 0; l < 2; l++) {   // records of surface l: slots (2v + l) RCAP + m, m < min(n, RCAP)
          const int ml = min(l ? (v ? n1B : n1A) : (v ? n0B : n0A), C2_RCAP);
          const float fl = l ? f1 : f0;
          macc *Gl = (v ? GB : GA) + (l ? N * 32 : 0);
#pragma unroll
          for (int m = 0; m < C2_RCAP; m++) {
            if (m >= ml) break;
            const float4 q = c2_recs[(2 * v + l) * C2_RCAP + m][threadIdx.x];
            const float wv = fl * q.w, u = q.y, vv = q.z, wa = wv * (1.f - u), wbb = wv * u;
            macc *pg = Gl + (__float_as_uint(q.x) << 5);
            atomicAdd(pg, q_raw(wa * (1.f - vv)));
            atomicAdd(pg + oy, q_raw(wbb * (1.f - vv)));
            atomicAdd(pg + 32, q_raw(wa * vv));
            atomicAdd(pg + oy + 32, q_raw(wbb * vv));
          }
        }
      }
      if (__any_sync(0xffffffffu, overA || overB)) {   // wide bands: re-walk, scatter crossings m >= RCAP
        int m0A = 0, m1A = 0, m0B = 0, m1B = 0, dd = 0;
        const int kend = __ldg(a.trav_off + rr + 1);
        float s_in0;
        const int k0 = band_entry_warp(a.trav, __ldg(a.trav_off + rr), kend, s_lo, s_in0);
        float Bd = 0.f, s = s_lo, za = s_lo * dz, ds = s_lo - s_in0;
        for (int k = k0; k < kend; k++) {
          const int2 w = __ldg(a.trav + k);
          const float4 cg = shift_geo(__ldg(a.trav_geo + k), ds);
          float2 km = C2_KMC ? make_float2(fmaf(cg.x, cg.w, cg.y * cg.z), cg.z * cg.w) : __ldg(a.trav_km + k);
          if (!C2_KMC) km.x = fmaf(2.f * km.y, ds, km.x);
          const float s1 = __int_as_float(w.y);
          const float zb = s1 * dz, Ls = s1 - s;
          const unsigned off = cell_off32(w.x);
#pragma unroll
          for (int l = 0; l < 2; l++) {
            const float zmin = l ? bd.z : bd.x, zmax = l ? bd.w : bd.y;
            if (zb <= zmin || za >= zmax) continue;
            const float4 *p = H4 + (size_t)l * N * 32 + off;
            const float4 r0 = __ldg(p), r1 = __ldg(p + oy);
            if (overA && (l ? n1A : n0A) > C2_RCAP)
              c2_cell<0, true>(r0.x, r0.y, r1.x, r1.y, cg, km, za, zb, Ls, dz, 0.f, Bd, l ? m1A : m0A, dd, nullptr,
                               GA + (l ? N * 32 : 0) + (off), oy, l ? f1A : f0A);
            if (overB && (l ? n1B : n0B) > C2_RCAP)
              c2_cell<0, true>(r0.z, r0.w, r1.z, r1.w, cg, km, za, zb, Ls, dz, 0.f, Bd, l ? m1B : m0B, dd, nullptr,
                               GB + (l ? N * 32 : 0) + (off), oy, l ? f1B : f0B);
          }
          if (s1 >= s_hi) break;
          s = s1;
          za = zb;
          ds = 0.f;
        }
      }
    } else {
#pragma unroll
      for (int v = 0; v < 2; v++) {
        if (v ? (dB || !actB) : (dA || !actA)) continue;
        const float b0 = v ? B0B : B0A, b1 = v ? B1B : B1A;
        const int64_t o = (int64_t)(v ? cB : cA) * a.R + __ldg(a.perm + rr);
        a.Lout[3 * o + 0] = b0;
        a.Lout[3 * o + 1] = b1 - b0;
        a.Lout[3 * o + 2] = s_exit - b1;
        a.Oout[o] = a.tc.k0 * b0 + a.tc.k1 * b1 + a.obase[rr];
      }
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(C2_THREADS, C2_MINB) k_trace_c2(TraceArgs a) {
  int N = a.tc.N, oy = a.tc.ny * 32;
  asm volatile("" : "+r"(N), "+r"(oy));   // keep in registers (no per-use reload / recompute)
  const int lane = threadIdx.x & 31;
  const int lin = blockIdx.y * gridDim.x + blockIdx.x, G2 = gridDim.y;
  const int tile = lin / (G2 * C2_TILE), within = lin - tile * (G2 * C2_TILE);
  const int g = within / C2_TILE, chunk = tile * C2_TILE + (within - (within / C2_TILE) * C2_TILE);
  const int cA = g * 64 + lane, cB = cA + 32;
  int acts = (cA < a.C ? 1 : 0) | (cB < a.C ? 2 : 0);
  asm volatile("" : "+r"(acts));
  const bool actA = acts & 1, actB = acts & 2;
  // lane-union band of its two chains per surface; the warp walks the union over 64 chains
  float4 bd = make_float4(3.0e38f, -3.0e38f, 3.0e38f, -3.0e38f);
  if (actA) bd = __ldg(a.band + cA);
  if (actB) {
    const float4 b = __ldg(a.band + cB);
    bd = make_float4(fminf(bd.x, b.x), fmaxf(bd.y, b.y), fminf(bd.z, b.z), fmaxf(bd.w, b.w));
  }
  float zlo = bd.x, zhi = bd.w;
  for (int o = 16; o > 0; o >>= 1) {
    zlo = fminf(zlo, __shfl_xor_sync(0xffffffffu, zlo, o));
    zhi = fmaxf(zhi, __shfl_xor_sync(0xffffffffu, zhi, o));
  }
  if (!actA && !actB) bd = make_float4(-3.0e38f, -3.0e38f, -3.0e38f, -3.0e38f);
  const float4 *__restrict__ H4 = reinterpret_cast<const float4 *>(a.cl) + (size_t)g * 2 * N * 32 + lane;
  asm volatile("mov.b64 %0, %0;" : "+l"(H4));
  float sllA = 0.f, sllB = 0.f;
  if (g * 64 + 64 <= a.C) c2_rays<MODE, true>(a, N, oy, g, chunk, acts, bd, zlo, zhi, H4, sllA, sllB);
  else c2_rays<MODE, false>(a, N, oy, g, chunk, acts, bd, zlo, zhi, H4, sllA, sllB);
  if (MODE == TRACE_LL) {
    if (actA) atomicAdd(a.ll + cA, q_ll(sllA));
    if (actB) atomicAdd(a.ll + cB, q_ll(sllB));
  }
}

// The chain x ray pairs the trace kernels deferred (an ill-conditioned cell,
// or more than RCAP crossings of a surface).  A group of DG lanes takes
// one pair, lane = one stored cell of its band (DG cells per round): the same fp32 cell code with
// the same cell pieces as the serial walk, ill-conditioned cells re-solved in
// place in fp64 from H + Hlo (HP2 lever 1), the lengths summed over the lanes,
// then the epilogue and each lane's adjoint scatter (or the path-length
// export).  A pair's latency is a few dependent loads, not a serial march.
// The last block resets the queue.
#ifndef DEFER_MINB
#define DEFER_MINB 2   // resident blocks per SM of k_trace_defer (launch bound and grid)
#endif
template <int MODE, int DG>
__global__ void __launch_bounds__(MT_THREADS, DEFER_MINB) k_trace_defer(TraceArgs a) {
  __shared__ float4 wrec[MT_THREADS][4];   // per lane: up to 2 crossings per surface of its cell
  load_geometry(a);
  __syncthreads();
  const int n = *(volatile int *)a.ovf_n;
  const int N = a.tc.N, ny = a.tc.ny;
  const int lane = threadIdx.x & (DG - 1), nq = min(n, a.ovf_cap);
  const unsigned gmask = DG == 32 ? 0xffffffffu : ((1u << DG) - 1u) << (threadIdx.x & 31 & ~(DG - 1));   // this group's lanes
  const int grp_g = (blockIdx.x * blockDim.x + threadIdx.x) / DG, ngrp = (gridDim.x * blockDim.x) / DG;
  int c_acc = -1;
  macc ll_acc = 0;   // fixed point per pair (R30): the sum does not depend on the queue order
  // one pair per group of DG lanes (all shuffles / ballots below are group-masked)
  auto process = [&](const int c, const int rr, const float s_lo, const float s_hi) {
    const Ray r = load_ray(a.ray_a, a.ray_b, rr);
    const size_t off = (size_t)(c >> 5) * 2 * N * 32 + (c & 31);
    const float *Hk = a.H + off, *Hl = a.Hlo + off;
    const float4 bd = a.band[c];
    float B0 = 0.f, B1 = 0.f;                          // this lane's cells' contributions
    int nr0 = 0, nr1 = 0, ovf = 0;
    if (s_lo < r.s_exit) {
      const int kend = a.trav_off[rr + 1];
      float s_in0;
      const int k0 = band_entry(a.trav, a.trav_off[rr], kend, s_lo, s_in0);
      float s_prev = s_lo;                             // s_out before this round's first cell
      for (int kb = k0; kb < kend; kb += DG) {
        const int k = kb + lane;
        const int2 w = k < kend ? __ldg(a.trav + k) : make_int2(0, __float_as_int(3.0e38f));
        const float s1 = __int_as_float(w.y);
        const float sp = __shfl_up_sync(gmask, s1, 1, DG);
        const float s = lane == 0 ? s_prev : sp;       // the piece [s, s1] of the serial walk
        const bool act = k < kend && s < s_hi;         // the walk stops after the cell reaching s_hi
        if (act) {
          const float4 cg = shift_geo(__ldg(a.trav_geo + k), k == k0 ? s_lo - s_in0 : 0.f);
          const int i = cell_i(w.x), j = cell_j(w.x), base = i * ny + j;
          const float za = s * r.dz, zb = s1 * r.dz, Ls = s1 - s;
#pragma unroll
          for (int l = 0; l < 2; l++) {
            const float zmin = l ? bd.z : bd.x, zmax = l ? bd.w : bd.y;
            float &B = l ? B1 : B0;
            int &nr = l ? nr1 : nr0;
            if (zb <= zmin) { B += Ls; continue; }
            if (za >= zmax) continue;
            const float *p = Hk + ((size_t)l * N + base) * 32;
            const float h00 = __ldg(p), h10 = __ldg(p + ny * 32), h01 = __ldg(p + 32), h11 = __ldg(p + ny * 32 + 32);
            if (zb <= fminf(fminf(h00, h10), fminf(h01, h11))) { B += Ls; continue; }
            if (za >= fmaxf(fmaxf(h00, h10), fmaxf(h01, h11))) continue;
            auto emit = [&](float u, float v, float ig) {
              if (nr < 2) wrec[threadIdx.x][2 * l + nr] = make_float4(__int_as_float(base), u, v, ig);
              else ovf = 1;
              nr++;
            };
            if (!solve32(h00, h10, h01, h11, cg, za, Ls, r.dz, B, emit)) {
              const float *pl = Hl + ((size_t)l * N + base) * 32;
              double se, se1;
              piece64(a, r, k, a.trav_off[rr], kend, k0, s_lo, se, se1);
              const Fix x = fix64((double)h00 + pl[0], (double)h10 + pl[ny * 32], (double)h01 + pl[32],
                                  (double)h11 + pl[ny * 32 + 32], sgeo[0][i], sgeo[0][i + 1], sgeo[1][j],
                                  sgeo[1][j + 1], r, se, se1);
              B += x.below;
              for (int m = 0; m < x.n; m++) emit(x.u[m], x.v[m], x.ig[m]);
            }
          }
        }
        // continue while this round's last cell ends below s_hi
        const float last = __shfl_sync(gmask, s1, DG - 1, DG);
        if (__ballot_sync(gmask, k < kend && s1 >= s_hi) || kb + DG >= kend) break;
        s_prev = last;   // (records accumulate over rounds: at most 2 per surface per lane, else ovf)
      }
    }
    // pair totals
    float T0 = B0, T1 = B1;
    for (int o = DG / 2; o > 0; o >>= 1) {
      T0 += __shfl_xor_sync(gmask, T0, o, DG);
      T1 += __shfl_xor_sync(gmask, T1, o, DG);
    }
    T0 += s_lo;
    T1 += s_lo;
    const bool anyovf = __ballot_sync(gmask, ovf) != 0;
    if (MODE == TRACE_LL) {
      float dldO;
      const float ll = epilogue(r.tb, r.cnt, a.tc, T0, T1, dldO);
      if (lane == 0) {
        if (c != c_acc) {
          if (c_acc >= 0) atomicAdd(a.ll + c_acc, ll_acc);
          c_acc = c;
          ll_acc = 0;
        }
        ll_acc += q_ll(ll);
      }
      const float f0 = dldO * a.tc.k0 * (float)MT_GQ, f1 = dldO * a.tc.k1 * (float)MT_GQ;
      if (!anyovf) {
        macc *G0 = a.G + off;
        for (int m = 0; m < nr0; m++) {
          const float4 t = wrec[threadIdx.x][m];
          scatter4(G0, 32, __float_as_int(t.x), ny, f0 * t.w, t.y, t.z);
        }
        for (int m = 0; m < nr1; m++) {
          const float4 t = wrec[threadIdx.x][2 + m];
          scatter4(G0 + (size_t)N * 32, 32, __float_as_int(t.x), ny, f1 * t.w, t.y, t.z);
        }
      } else if (lane == 0 && s_lo < r.s_exit) {
        // rare: a lane with more than 2 crossings of a surface over its cells (bands of
        // more than DG cells): one lane re-walks and scatters directly
        float s_in0, d0 = s_lo, d1 = s_lo;
        int nrec[2] = {0, 0};
        const int kend = a.trav_off[rr + 1];
        const int k0 = band_entry(a.trav, a.trav_off[rr], kend, s_lo, s_in0);
        walk<32, true>(&a, a.trav_off[rr], r, a.trav, a.trav_geo, k0, kend, s_lo, s_in0, s_hi, ny, N, Hk, Hl, a.G + off, bd,
                       d0, d1, nullptr, nrec, f0, f1);
      }
    } else if (lane == 0) {
      const int64_t o = (int64_t)c * a.R + a.perm[rr];
      a.Lout[3 * o + 0] = T0;
      a.Lout[3 * o + 1] = T1 - T0;
      a.Lout[3 * o + 2] = r.s_exit - T1;
      a.Oout[o] = a.tc.k0 * T0 + a.tc.k1 * T1 + a.obase[rr];
    }
  };
  // the queued pairs (walk range as queued: the warp's union band)
  for (int q = grp_g; q < nq; q += ngrp) {
    const float4 e0 = a.ovf_q[q];
    process(__float_as_int(e0.x), __float_as_int(e0.y), e0.z, e0.w);
  }
  // queue overflow: the pairs that did not fit are marked in the (C x R)-bit redo
  // bitmap; walk range = the pair's own chain band (a subset of the union band
  // the main kernel would have used: the same lengths up to rounding)
  if (n > a.ovf_cap) {
    const int64_t nw = ((int64_t)a.C * a.R + 31) / 32;
    for (int64_t wi = grp_g; wi < nw; wi += ngrp) {
      unsigned bits = a.redo[wi];
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1u;
        const int64_t idx = wi * 32 + b;
        const int c = (int)(idx / a.R), rr = (int)(idx - (int64_t)c * a.R);
        const float4 bd = a.band[c];
        const float2 rb = __ldg(reinterpret_cast<const float2 *>(a.ray_b + rr));
        process(c, rr, fminf(__fdividef(bd.x, rb.x) * (1.f - 1e-6f), rb.y),
                fminf(__fdividef(bd.w, rb.x) * (1.f + 1e-6f), rb.y));
      }
      __syncwarp(gmask);
      if (lane == 0 && a.redo[wi]) a.redo[wi] = 0u;
    }
  }
  if (MODE == TRACE_LL && lane == 0 && c_acc >= 0) atomicAdd(a.ll + c_acc, ll_acc);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(a.ovf_done, 1) == (int)gridDim.x - 1) {
      *a.ovf_total += (unsigned long long)n;
      *a.ovf_n = 0;
      *a.ovf_done = 0;
    }
  }
}

// ---------------------------------------------------------------------------
// K2, ray lanes (small C, e.g. the single-chain ray-sharded config): block row
// = one chain whose heights ([2N] fp32, 32 KiB at n = 64) sit in shared
// memory; thread = ray (rays Morton-ordered, so a warp's rays walk nearby
// cells).  Same cell code as the chain lanes; ill-conditioned pairs and pairs
// with more than RCAP crossings of a surface go to k_trace_defer; the adjoint
// is a RED.ADD.F32 per corner into the chain's ∂ℓ/∂H column (shared-memory
// fp32 atomics are CAS loops on sm_100a).
// ---------------------------------------------------------------------------
template <int MODE, int NY>
__global__ void __launch_bounds__(MT_THREADS, MT_RL_MINB) k_trace_rl(TraceArgs a, const float *__restrict__ Hc) {
  extern __shared__ __align__(16) float smem[];
  __shared__ macc red[MT_THREADS / 32];
  const int ny = NY ? NY : a.tc.ny, N = a.tc.N;
  const int tid = threadIdx.x, c = blockIdx.y;
#if MT_RL_GLOBAL_H
  // the chain's heights straight from global memory (L1-resident: 2N floats);
  // shared memory holds only the crossing records, so more blocks fit per SM
  const float *__restrict__ Hs = Hc + (size_t)c * 2 * N;
  float4 *rec = reinterpret_cast<float4 *>(smem) + tid;                        // [2*RCAP][MT_THREADS]
#else
  float *Hs = smem;                                                            // [2N]
  float4 *rec = reinterpret_cast<float4 *>(smem + ((2 * N + 3) & ~3)) + tid;   // [2*RCAP][MT_THREADS]
  {
    const float *src = Hc + (size_t)c * 2 * N;
    for (int k = tid; k < 2 * N; k += MT_THREADS) Hs[k] = __ldg(src + k);
  }
#endif
  load_geometry(a);
  const float4 bd = __ldg(a.band + c);
  const size_t coff = (size_t)(c >> 5) * 2 * N * 32 + (c & 31);
  macc *G0 = a.G + coff;
  __shared__ int next_ray;
  const int r_begin = blockIdx.x * (int)a.rays_per_block;
  const int r_end = min((int)a.R, r_begin + (int)a.rays_per_block);
  if (tid == 0) next_ray = r_begin;
  __syncthreads();
  macc llacc = 0;   // fixed point per pair (R30): independent of which warp took which rays
  const int lane = tid & 31;
  // warps take 32 consecutive (Morton-adjacent) rays at a time from the block's range:
  // thread-serial walks vary in length, and a static split left warps idle at the end
  long long t_task = 0;
  int prev_base = -1;
  for (;;) {
    int base = 0;
    if (lane == 0) base = atomicAdd(&next_ray, 32);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (a.task_cost && lane == 0) {   // measurement mode (mt_ray_cost): SM cycles of each 32-ray task
      const long long t = clock64();
      if (prev_base >= 0) a.task_cost[prev_base >> 5] = (unsigned long long)(t - t_task);
      t_task = t;
      prev_base = base;
    }
    if (base >= r_end) break;
    const int rr = base + lane;
    if (rr >= r_end) continue;
    const float2 rb = __ldg(reinterpret_cast<const float2 *>(a.ray_b + rr));
    const float dz = rb.x, s_exit = rb.y;
    const float s_lo = fminf(__fdividef(bd.x, dz) * (1.f - 1e-6f), s_exit);
    const float s_hi = fminf(__fdividef(bd.w, dz) * (1.f + 1e-6f), s_exit);
    float B0 = s_lo, B1 = s_lo;
    int n0 = 0, n1 = 0, defer = 0;
    if (s_lo < s_exit) {
      // replay of the exact traversal from 2-bit exit codes (a2): the exit parameter
      // of each cell is recomputed with the builder's fp32 operations, so the cells
      // and their pieces are bit-identical to the stored traversal, from 16 B/ray
      // of coalesced, L2-resident codes instead of 8 B/cell of scattered lists
      const int2 hd = __ldg(a.rl_head + rr);
      const uint4 cw = __ldg(a.rl_code + rr);
      const int ncell = hd.x & 255;
      int i = (hd.x >> 8) & 127, j = (hd.x >> 15) & 127;
      const float2 ro = __ldg(reinterpret_cast<const float2 *>(a.ray_a + rr));
      const float2 rd = __ldg(reinterpret_cast<const float2 *>(a.ray_a + rr) + 1);
      const int sx = rd.x > 0.f ? 1 : (rd.x < 0.f ? -1 : 0), sy = rd.y > 0.f ? 1 : (rd.y < 0.f ? -1 : 0);
      const float adx = fabsf(rd.x), ady = fabsf(rd.y);
      const float iadx = adx > 0.f ? 1.f / adx : 0.f, iady = ady > 0.f ? 1.f / ady : 0.f;
      float s_prev = 0.f, s = s_lo, za = s_lo * dz;
      int k = 0;
      // jump to the band: the cell holding s_lo is (i, j) -> list entry |Δi| + |Δj| when no
      // vertex step precedes it; checked against the codes (x/y step counts) and the
      // recomputed exit parameters, else the replay simply starts from the first cell
      if (ncell <= 64) {
        const float x = fmaf(s_lo, rd.x, ro.x), y = fmaf(s_lo, rd.y, ro.y);
        const int nx = a.tc.nx;
        int ie = min(max((int)((x - sgeo[0][0]) * ((float)(nx - 1) / (sgeo[0][nx - 1] - sgeo[0][0]))), 0), nx - 2);
        int je = min(max((int)((y - sgeo[1][0]) * ((float)(ny - 1) / (sgeo[1][ny - 1] - sgeo[1][0]))), 0), ny - 2);
        while (ie < nx - 2 && sgeo[0][ie + 1] <= x) ie++;
        while (ie > 0 && sgeo[0][ie] > x) ie--;
        while (je < ny - 2 && sgeo[1][je + 1] <= y) je++;
        while (je > 0 && sgeo[1][je] > y) je--;
        const int ke = abs(ie - i) + abs(je - j);
        if (ke > 1 && ke < ncell) {
          // x and y steps among the exits of cells 0 .. ke-2 (the ones before cell ke-1)
          const int m = ke - 1;
          int nxs = 0, nys = 0;
#pragma unroll
          for (int q = 0; q < 4; q++) {
            const uint32_t wq = q == 0 ? cw.x : (q == 1 ? cw.y : (q == 2 ? cw.z : cw.w));
            const int lo = 16 * q, cnt = min(max(m - lo, 0), 16);
            const uint32_t mask = cnt >= 16 ? 0xffffffffu : ((1u << (2 * cnt)) - 1u);
            nxs += __popc(wq & mask & 0x55555555u);
            nys += __popc(wq & mask & 0xaaaaaaaau);
          }
          const int ip = i + sx * nxs, jp = j + sy * nys;    // cell ke-1
          if (nxs + nys == m) {                               // no vertex step before it
            const uint32_t wp = m - 1 < 16 ? cw.x : (m - 1 < 32 ? cw.y : (m - 1 < 48 ? cw.z : cw.w));
            const int cp = (wp >> (2 * ((m - 1) & 15))) & 3;   // exit code of cell ke-2
            // exit parameter of cell ke-2 (its stored s_out) needs that cell's (i, j)
            const int i2 = ip - ((cp & 1) ? sx : 0), j2 = jp - ((cp & 2) ? sy : 0);
            float e2;
            if (cp == 0) e2 = s_exit;
            else if (cp & 1) e2 = __fmul_rn(sx > 0 ? __fsub_rn(sgeo[0][i2 + 1], ro.x) : __fsub_rn(ro.x, sgeo[0][i2]), iadx);
            else e2 = __fmul_rn(sy > 0 ? __fsub_rn(sgeo[1][j2 + 1], ro.y) : __fsub_rn(ro.y, sgeo[1][j2]), iady);
            const float sp2 = fminf(e2, s_exit);
            if (sp2 <= s_lo) {   // cells before ke-1 end at or below s_lo: start the replay at ke-1
              k = m;
              i = ip;
              j = jp;
              s_prev = sp2;      // (monotone s_out: max with earlier values is a no-op here)
            }
          }
        }
      }
      // branch-free exit parameter: next x-line X[i + px] (px = [d_x > 0]) at distance
      // sx·(X - o_x) (exact, HP3) over |d_x|; likewise y; code 0 = the top exit
      const int px = sx > 0, py = sy > 0;
      const float sxf = (float)sx, syf = (float)sy;
      uint32_t word = k < 64 ? (k < 32 ? (k < 16 ? cw.x : cw.y) : (k < 48 ? cw.z : cw.w))
                             : __ldg(a.rl_ovf + hd.y + ((k - 64) >> 4));
      word >>= 2 * (k & 15);
      for (; k < ncell; k++) {
        if (k > 0 && (k & 15) == 0)
          word = k < 64 ? (k == 16 ? cw.y : (k == 32 ? cw.z : cw.w)) : __ldg(a.rl_ovf + hd.y + ((k - 64) >> 4));
        const int code = word & 3;
        word >>= 2;
        const float numx = __fmul_rn(__fsub_rn(sgeo[0][i + px], ro.x), sxf);
        const float numy = __fmul_rn(__fsub_rn(sgeo[1][j + py], ro.y), syf);
        const float s_ev = code == 0 ? s_exit : __fmul_rn((code & 1) ? numx : numy, (code & 1) ? iadx : iady);
        const float s1 = fmaxf(fminf(s_ev, s_exit), s_prev);   // the stored s_out
        if (s1 > s_lo) {                                         // in the band (from its entry cell on)
          const float ix = sgeo[2][i], iy = sgeo[3][j];
          const float4 cg = make_float4((fmaf(s, rd.x, ro.x) - sgeo[0][i]) * ix,
                                        (fmaf(s, rd.y, ro.y) - sgeo[1][j]) * iy, rd.x * ix, rd.y * iy);
          const float zb = s1 * dz, Ls = s1 - s;
          const int base = i * ny + j, w = base << 5;
          // the ray-only solve terms K = u0 β + v0 α, M = α β of solve32k (the chain lanes store them)
          const float2 km = RL_KM ? make_float2(fmaf(cg.x, cg.w, cg.y * cg.z), cg.z * cg.w) : make_float2(0.f, 0.f);
          if (zb <= bd.x) B0 += Ls;
          else if (za < bd.y) {
            const float *p = Hs + base;
            cw_solve<0, RL_KM>(make_float4(p[0], p[1], p[ny], p[ny + 1]), w, cg, za, zb, Ls, dz, B0, n0, defer, rec, km);
          }
          if (zb <= bd.z) B1 += Ls;
          else if (za < bd.w) {
            const float *p = Hs + N + base;
            cw_solve<1, RL_KM>(make_float4(p[0], p[1], p[ny], p[ny + 1]), w, cg, za, zb, Ls, dz, B1, n1, defer, rec, km);
          }
          if (s1 >= s_hi) break;
          s = s1;
          za = zb;
        }
        if (code & 1) i += sx;
        if (code & 2) j += sy;
        s_prev = s1;
      }
    }
    if (defer || n0 > RCAP || n1 > RCAP) {             // rare: the whole pair goes to k_trace_defer
      const int q = atomicAdd(a.ovf_n, 1);
      if (q < a.ovf_cap) a.ovf_q[q] = make_float4(__int_as_float(c), __int_as_float(rr), s_lo, s_hi);
      else redo_mark(a, c, rr);   // queue full: the follow-up kernel finds the pair in the bitmap
      continue;
    }
    if (MODE == TRACE_LL) {
      const float2 rt = __ldg(reinterpret_cast<const float2 *>(a.ray_b + rr) + 1);
      float dldO;
      llacc += q_ll(epilogue(rt.x, rt.y, a.tc, B0, B1, dldO));
      const float f0 = dldO * a.tc.k0 * (float)MT_GQ, f1 = dldO * a.tc.k1 * (float)MT_GQ;
      if (fmaxf(fabsf(f0), fabsf(f1)) * (1.f / GTHR) < MT_QSMALL)
        scatter_recs<true>(rec, n0, n1, G0, N, ny * 32, f0, f1);
      else
        scatter_recs<false>(rec, n0, n1, G0, N, ny * 32, f0, f1);
    } else {
      const int64_t o = (int64_t)c * a.R + __ldg(a.perm + rr);
      a.Lout[3 * o + 0] = B0;
      a.Lout[3 * o + 1] = B1 - B0;
      a.Lout[3 * o + 2] = s_exit - B1;
      a.Oout[o] = a.tc.k0 * B0 + a.tc.k1 * B1 + a.obase[rr];
    }
  }
  if (MODE == TRACE_LL) {
    macc v = llacc;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((tid & 31) == 0) red[tid >> 5] = v;
    __syncthreads();
    if (tid == 0) {
      macc t = 0;
      for (int w = 0; w < MT_THREADS / 32; w++) t += red[w];
      atomicAdd(a.ll + c, t);
    }
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
static TraceArgs base_trace_args(mt_problem *p) {
  TraceArgs a{};
  a.tc = p->tc;
  a.X = p->d_X; a.Y = p->d_Y;
  a.ray_a = p->d_ray_a; a.ray_b = p->d_ray_b; a.obase = p->d_obase;
  a.trav_off = p->d_trav_off; a.trav = p->d_trav; a.trav_geo = p->d_trav_geo; a.trav_km = p->d_trav_km;
  a.rl_head = p->d_rl_head; a.rl_code = p->d_rl_code; a.rl_ovf = p->d_rl_ovf;
  a.perm = p->d_perm;
  a.R = p->R;
  a.ovf_q = p->d_ovf_q; a.ovf_n = p->d_ovf_n; a.ovf_done = p->d_ovf_n + 1; a.ovf_cap = p->ovf_cap;
  a.redo = p->d_redo;
  a.ovf_total = reinterpret_cast<unsigned long long *>(p->d_ovf_n + 2);
  return a;
}

cudaError_t build_traversal(mt_problem *p) {
  if (p->R <= 0) return cudaSuccess;
  TraceArgs a = base_trace_args(p);
  int32_t *d_cnt = nullptr;
  cudaError_t e = cudaMalloc(&d_cnt, sizeof(int32_t) * p->R);
  if (e != cudaSuccess) return e;
  unsigned nb = (unsigned)((p->R + 127) / 128);
  k_build_trav<<<nb, 128>>>(a, nullptr, d_cnt, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
  std::vector<int32_t> cnt(p->R);
  e = cudaMemcpy(cnt.data(), d_cnt, sizeof(int32_t) * p->R, cudaMemcpyDeviceToHost);
  cudaFree(d_cnt);
  if (e != cudaSuccess) return e;
  std::vector<int32_t> off(p->R + 1, 0), ovf(p->R + 1, 0);
  int64_t tot = 0;
  for (int64_t q = 0; q < p->R; q++) {
    tot += cnt[q];
    if (tot >= (int64_t)1 << 31) return cudaErrorInvalidValue;   // > 2^31 stored cells
    off[q + 1] = (int32_t)tot;
    ovf[q + 1] = ovf[q] + (cnt[q] > 64 ? (cnt[q] - 64 + 15) / 16 : 0);   // step-code words past 64 cells
  }
  p->trav_cells = tot;
  e = cudaMalloc(&p->d_trav_off, sizeof(int32_t) * (p->R + 1));
  const size_t ncells = p->trav_cells > 0 ? p->trav_cells : 1;
  if (e == cudaSuccess) e = cudaMalloc(&p->d_trav, sizeof(int2) * ncells);
  if (e == cudaSuccess) e = cudaMalloc(&p->d_trav_geo, sizeof(float4) * ncells);
  if (e == cudaSuccess) e = cudaMalloc(&p->d_trav_km, sizeof(float2) * ncells);
  if (e == cudaSuccess) e = cudaMalloc(&p->d_rl_head, sizeof(int2) * p->R);
  if (e == cudaSuccess) e = cudaMalloc(&p->d_rl_code, sizeof(uint4) * p->R);
  if (e == cudaSuccess) e = cudaMalloc(&p->d_rl_ovf, sizeof(uint32_t) * (ovf[p->R] > 0 ? ovf[p->R] : 1));
  int32_t *d_ovfoff = nullptr;
  if (e == cudaSuccess) e = cudaMalloc(&d_ovfoff, sizeof(int32_t) * (p->R + 1));
  if (e == cudaSuccess) e = cudaMemcpy(d_ovfoff, ovf.data(), sizeof(int32_t) * (p->R + 1), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(p->d_rl_ovf, 0, sizeof(uint32_t) * (ovf[p->R] > 0 ? ovf[p->R] : 1));
  if (e == cudaSuccess)
    e = cudaMemcpy(p->d_trav_off, off.data(), sizeof(int32_t) * (p->R + 1), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return e;
  a.trav_off = p->d_trav_off;
  a.trav = p->d_trav;
  a.trav_geo = p->d_trav_geo;
  a.trav_km = p->d_trav_km;
  if (e == cudaSuccess)
    k_build_trav<<<nb, 128>>>(a, p->d_trav_off, nullptr, p->d_trav, p->d_trav_geo, p->d_trav_km, p->d_rl_head,
                              p->d_rl_code, p->d_rl_ovf, d_ovfoff);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  cudaFree(d_ovfoff);
  return e;
}

template <typename Kern>
static cudaError_t set_smem(Kern k, size_t smem, size_t *done) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (smem > 32 * 1024 && done[dev & 15] < smem) {   // (dynamic + static must fit the attribute)
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    done[dev & 15] = smem;
  }
  return cudaSuccess;
}

template <int MODE, int NY>
static cudaError_t launch_v0(const TraceArgs &a, dim3 grid, cudaStream_t s) {
  k_trace_v0<MODE, NY><<<grid, MT_THREADS, (size_t)16 * 2 * RCAP * MT_THREADS, s>>>(a);
  return cudaGetLastError();
}

template <int MODE>
static cudaError_t launch_v0_ny(const TraceArgs &a, int ny, dim3 grid, cudaStream_t s) {
  switch (ny) {
    case 8: return launch_v0<MODE, 8>(a, grid, s);
    case 16: return launch_v0<MODE, 16>(a, grid, s);
    case 32: return launch_v0<MODE, 32>(a, grid, s);
    case 64: return launch_v0<MODE, 64>(a, grid, s);
    default: return launch_v0<MODE, 0>(a, grid, s);
  }
}

#ifndef C2_CARVE
#define C2_CARVE -2   // shared-memory carveout (percent) of k_trace_c2; -2: just enough for C2_MINB blocks
#endif
template <int MODE>
static cudaError_t launch_c2(const TraceArgs &a, dim3 grid, cudaStream_t s) {
  // The records are the kernel's only shared memory; the rest of the SM's 256 KB serves
  // as L1 for the corner loads, and a carveout sized to the resident blocks (100 KB
  // instead of the driver's 164 KB) raises the L1 hit rate 52 -> 59% (-5% trace time).
  if (C2_CARVE != -1) {
    static bool done[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!done[dev & 63]) {
      int pct = C2_CARVE;
      if (pct < 0) {
        cudaFuncAttributes fa;
        int mx = 0;
        cudaError_t e = cudaFuncGetAttributes(&fa, k_trace_c2<MODE>);
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&mx, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        if (e != cudaSuccess) return e;
        const long need = (long)C2_MINB * ((long)fa.sharedSizeBytes + 1024);   // + 1 KB reserved per block
        pct = (int)std::min<long>(100, (need * 100 + mx - 1) / std::max(mx, 1));
      }
      cudaError_t e = cudaFuncSetAttribute(k_trace_c2<MODE>, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
      if (e != cudaSuccess) return e;
      done[dev & 63] = true;
    }
  }
  k_trace_c2<MODE><<<grid, C2_THREADS, 0, s>>>(a);   // (records in static shared memory)
  return cudaGetLastError();
}


template <int MODE, int NY>
static cudaError_t launch_rl(const TraceArgs &a, const float *Hc, dim3 grid, size_t smem, cudaStream_t s) {
  static size_t done[16] = {0};
  cudaError_t e = set_smem(k_trace_rl<MODE, NY>, smem, done);
  if (e != cudaSuccess) return e;
  k_trace_rl<MODE, NY><<<grid, MT_THREADS, smem, s>>>(a, Hc);
  return cudaGetLastError();
}

template <int MODE>
static cudaError_t launch_rl_ny(const TraceArgs &a, const float *Hc, int ny, dim3 grid, size_t smem,
                                cudaStream_t s) {
  switch (ny) {
    case 8: return launch_rl<MODE, 8>(a, Hc, grid, smem, s);
    case 16: return launch_rl<MODE, 16>(a, Hc, grid, smem, s);
    case 32: return launch_rl<MODE, 32>(a, Hc, grid, smem, s);
    case 64: return launch_rl<MODE, 64>(a, Hc, grid, smem, s);
    default: return launch_rl<MODE, 0>(a, Hc, grid, smem, s);
  }
}

cudaError_t launch_trace(mt_problem *p, int mode, int C, const float *H, const float4 *band,
                         macc *G, macc *ll, float *L, float *O, cudaStream_t s, unsigned long long *task_cost) {
  if (C <= 0 || p->R <= 0) return cudaSuccess;
  if (mode == TRACE_LL && p->vx.nz > 0) return launch_voxel(p, C, H, band, G, ll, s);   // f3 model active
  TraceArgs a = base_trace_args(p);
  a.C = C;
  a.H = H; a.Hlo = p->d_Hlo; a.band = band; a.G = G; a.ll = ll; a.Lout = L; a.Oout = O;
  a.task_cost = task_cost;
  const bool chain_lanes = p->trace_k == 0 ? C >= 16 : p->trace_k == 32;
  cudaError_t e = cudaSuccess;
  bool rec = p->timing && p->n_rec < (int)p->ev_a.size();
  if (rec) cudaEventRecord(p->ev_a[p->n_rec], s);
  if (chain_lanes) {
    int groups = (C + 31) / 32;
    const bool c2 = p->cl_v == 2 || (p->cl_v < 0 && C >= 64);
    if (c2) {   // two chains per lane: paired heights of both chains
      const int64_t n = (int64_t)((C + 63) / 64) * 2 * p->N * 32;
      k_cell_prep2<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(H, reinterpret_cast<float4 *>(p->d_cl), C, p->ny,
                                                             p->N, n);
      p->all_launches++;
    } else {   // paired heights (H(i,j), H(i,j+1))
      const int64_t n = (int64_t)groups * 2 * p->N * 32;
      k_cell_prep<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(H, reinterpret_cast<float2 *>(p->d_cl), p->ny, n);
      p->all_launches++;
    }
    a.cl = p->d_cl;
    // ray chunks of <= 512 Morton-ordered rays per block (compact, L1-friendly regions, many
    // waves for load balance).  The shape depends on R only, never on C, so a chain's
    // result is bit-identical whatever the chain count per GPU (R30, chain sharding).
    const int64_t chunk = p->chunk > 0 ? p->chunk
                                       : std::max<int64_t>(32, std::min<int64_t>(512, p->R / (2 * (int64_t)p->num_sms)));
    a.rays_per_block = chunk;
    int64_t S = (p->R + chunk - 1) / chunk;
    dim3 grid((unsigned)S, (unsigned)groups);
    if (c2) {
      // two chains per lane: R / (2.75 SMs) rays per 256-thread block, at most 512 (Small,
      // R = 16,384: 40-ray chunks, 0.0605 -> 0.0523 ms per evaluation vs R / (2 SMs); every
      // R >= 225K keeps 512).  Again a function of R (and the device) only, never of C.
      const int64_t chunk2 = p->chunk > 0 ? p->chunk
                                          : std::max<int64_t>(32, std::min<int64_t>(512, p->R * 4 / (11 * (int64_t)p->num_sms)));
      a.rays_per_block = std::max<int64_t>(32, chunk2 * C2_THREADS / 256);
      const int64_t S2 = (p->R + a.rays_per_block - 1) / a.rays_per_block;
      dim3 grid2((unsigned)S2, (unsigned)((C + 63) / 64));
      if (grid2.x % C2_TILE) grid2.x += C2_TILE - grid2.x % C2_TILE;   // whole tiles (extra chunks are empty)
      e = mode == TRACE_LL ? launch_c2<TRACE_LL>(a, grid2, s) : launch_c2<TRACE_PATH>(a, grid2, s);
    } else {
      e = mode == TRACE_LL ? launch_v0_ny<TRACE_LL>(a, p->ny, grid, s) : launch_v0_ny<TRACE_PATH>(a, p->ny, grid, s);
    }
    if (rec) cudaEventRecord(p->ev_m[p->n_rec], s);
    if (e == cudaSuccess) {   // deferred pairs (ill-conditioned or > RCAP crossings)
      // few rays -> few deferred pairs: the follow-up's time is one pair's chain of dependent
      // band rounds, so a whole warp per pair (Small: 16.5 -> 12.9 us per evaluation); a
      // function of R only, like the launch shape (R30)
      const dim3 gd(DEFER_MINB * p->num_sms);
      if (p->R <= DEFER_SMALL_R) {
        if (mode == TRACE_LL) k_trace_defer<TRACE_LL, 32><<<gd, MT_THREADS, 0, s>>>(a);
        else k_trace_defer<TRACE_PATH, 32><<<gd, MT_THREADS, 0, s>>>(a);
      } else if (mode == TRACE_LL) {
        k_trace_defer<TRACE_LL, DEFER_DG><<<gd, MT_THREADS, 0, s>>>(a);
      } else {
        k_trace_defer<TRACE_PATH, DEFER_DG><<<gd, MT_THREADS, 0, s>>>(a);
      }
      e = cudaGetLastError();
      p->all_launches++;
    }
  } else {
    // contiguous [C][2N] copy of the chains' heights for the shared-memory tiles
    e = launch_tile(p, C, H, p->d_Hc, 0, s);
    int64_t S = p->trace_s > 0 ? p->trace_s : std::max<int64_t>(1, (int64_t)p->num_sms * 4 * 4 / C);
    S = std::min<int64_t>(S, (p->R + 255) / 256);
    a.rays_per_block = (p->R + S - 1) / S;
    S = (p->R + a.rays_per_block - 1) / a.rays_per_block;
    dim3 grid((unsigned)S, (unsigned)C);
    size_t smem = (MT_RL_GLOBAL_H ? 0 : (size_t)4 * ((2 * p->N + 3) & ~3)) + (size_t)16 * 2 * RCAP * MT_THREADS;
    if (e == cudaSuccess)
      e = mode == TRACE_LL ? launch_rl_ny<TRACE_LL>(a, p->d_Hc, p->ny, grid, smem, s)
                           : launch_rl_ny<TRACE_PATH>(a, p->d_Hc, p->ny, grid, smem, s);
    if (rec) cudaEventRecord(p->ev_m[p->n_rec], s);
    if (e == cudaSuccess) {
      if (p->R <= DEFER_SMALL_R) {
        if (mode == TRACE_LL) k_trace_defer<TRACE_LL, 32><<<2 * p->num_sms, MT_THREADS, 0, s>>>(a);
        else k_trace_defer<TRACE_PATH, 32><<<2 * p->num_sms, MT_THREADS, 0, s>>>(a);
      } else if (mode == TRACE_LL) {
        k_trace_defer<TRACE_LL, DEFER_DG_RL><<<2 * p->num_sms, MT_THREADS, 0, s>>>(a);
      } else {
        k_trace_defer<TRACE_PATH, DEFER_DG_RL><<<2 * p->num_sms, MT_THREADS, 0, s>>>(a);
      }
      e = cudaGetLastError();
      p->all_launches += 2;
    }
  }
  if (rec) { cudaEventRecord(p->ev_b[p->n_rec], s); p->n_rec++; }
  p->all_launches++;
  p->trace_launches++;
  p->pairs += (double)C * (double)p->R;
  return e;
}
