// Pseudo-acoustic TTI (two coupled fields p, r) for sm_100a.
//
// Replaces compute(box, equation) for the TTI family: the rotated operator
// G = D^T D of PAPER.md:1005-1018 / SPEC.md:594-601 expressed as nested
// first derivatives (radius SO; the reference's nested Deriv(coef*Deriv)
// lowering, symbolics.py:556-566), in Devito's centred two-field form:
//
//   g(f)   = a_x Dx f + a_y Dy f + a_z Dz f           (a = symmetry axis)
//   Gzz(f) = sum_i D_i (a_i g(f))
//   H0(p)  = L(p) - Gzz(p)
//   p1 = 2 p0 - p2 + dt2/m (epsp H0(p) + delp Gzz(r))
//   r1 = 2 r0 - r2 + dt2/m (delp H0(p) + Gzz(r))
//
// Two passes per box: pass 1 writes g(p), g(r) on the box grown by R into a
// FULL-shaped scratch pair; pass 2 applies the outer derivative and the
// update.  Each pass exists as a generic (one thread per point) and a TMA
// streaming (stream.cuh) launch sharing one per-point routine, so every
// launch geometry gives identical bits.
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"
#include "stream.cuh"

namespace sdmp {

struct TTICoef {
  float lap[3][SDMP_NCOEF];
  float d1[3][SDMP_NCOEF];
  float csum0;
  float dt2;
  int m_is_scale;  // the m operand already holds RN(dt2 / m) (bound by the plan)
};

// dt2 / m per point, or the bound scale (identical bits: __fdiv_rn both ways)
template <class T>
__device__ __forceinline__ T tti_scale(const TTICoef& c, T m) {
  return c.m_is_scale ? m : vdiv(vconst<T>(c.dt2), m);
}

// logical ids: tap fields and pointwise fields
enum { TP = 0, TR, TAX, TAY, TAZ, TGP, TGR, NT_ };
enum { QP2 = 0, QR0, QR2, QM, QE, QD, QAX, QAY, QAZ, NQ_ };

// All sums start from an explicit fma with a zero addend and products are
// folded into fmas, so no separately rounded product feeds an add (ptxas
// contracts packed mul+add): float and V2 evaluations give identical bits.
template <int R, int AX, int F, class A>
__device__ __forceinline__ typename A::T dcentral(const A& a, const float* w) {
  using T = typename A::T;
  T acc = vcfma(w[1], vsub(a.template t<F, AX>(1), a.template t<F, AX>(-1)), vconst<T>(0.f));
#pragma unroll
  for (int k = 2; k <= R; ++k)
    acc = vcfma(w[k], vsub(a.template t<F, AX>(k), a.template t<F, AX>(-k)), acc);
  return acc;
}

// D_AX (a_AX g) with a, g both tapped: term_k = a(k) g(k) - a(-k) g(-k)
// evaluated as fma(a(k), g(k), 0 - RN(a(-k) g(-k))).
template <int R, int AX, int FA, int FG, class A>
__device__ __forceinline__ typename A::T outer(const A& a, const float* w) {
  using T = typename A::T;
  T acc = vconst<T>(0.f);
#pragma unroll
  for (int k = 1; k <= R; ++k) {
    const T nlo = vnmul(a.template t<FA, AX>(-k), a.template t<FG, AX>(-k));
    const T term = vfma(a.template t<FA, AX>(k), a.template t<FG, AX>(k), nlo);
    acc = vcfma(w[k], term, acc);
  }
  return acc;
}

template <int R, class A>
__device__ __forceinline__ void g_point(const A& a, const TTICoef& c, typename A::T& gp,
                                        typename A::T& gr) {
  using T = typename A::T;
  const T ax = a.template q<QAX>(), ay = a.template q<QAY>(), az = a.template q<QAZ>();
  gp = vfma(ax, dcentral<R, 0, TP>(a, c.d1[0]), vconst<T>(0.f));
  gp = vfma(ay, dcentral<R, 1, TP>(a, c.d1[1]), gp);
  gp = vfma(az, dcentral<R, 2, TP>(a, c.d1[2]), gp);
  gr = vfma(ax, dcentral<R, 0, TR>(a, c.d1[0]), vconst<T>(0.f));
  gr = vfma(ay, dcentral<R, 1, TR>(a, c.d1[1]), gr);
  gr = vfma(az, dcentral<R, 2, TR>(a, c.d1[2]), gr);
}

template <int R, class A>
__device__ __forceinline__ void u_point(const A& a, const TTICoef& c, typename A::T& p1,
                                        typename A::T& r1) {
  using T = typename A::T;
  T gzp = outer<R, 0, TAX, TGP>(a, c.d1[0]);
  gzp = vadd(gzp, outer<R, 1, TAY, TGP>(a, c.d1[1]));
  gzp = vadd(gzp, outer<R, 2, TAZ, TGP>(a, c.d1[2]));
  T gzr = outer<R, 0, TAX, TGR>(a, c.d1[0]);
  gzr = vadd(gzr, outer<R, 1, TAY, TGR>(a, c.d1[1]));
  gzr = vadd(gzr, outer<R, 2, TAZ, TGR>(a, c.d1[2]));
  const T c0 = a.template t<TP, 0>(0);
  T lap = vcfma(c.csum0, c0, vconst<T>(0.f));
#pragma unroll
  for (int k = 1; k <= R; ++k)
    lap = vcfma(c.lap[0][k], vadd(a.template t<TP, 0>(-k), a.template t<TP, 0>(k)), lap);
#pragma unroll
  for (int k = 1; k <= R; ++k)
    lap = vcfma(c.lap[1][k], vadd(a.template t<TP, 1>(-k), a.template t<TP, 1>(k)), lap);
#pragma unroll
  for (int k = 1; k <= R; ++k)
    lap = vcfma(c.lap[2][k], vadd(a.template t<TP, 2>(-k), a.template t<TP, 2>(k)), lap);
  const T h0 = vsub(lap, gzp);
  const T sc = tti_scale(c, a.template q<QM>());
  const T e = a.template q<QE>(), d = a.template q<QD>();
  const T pp = vfma(d, gzr, vmul(e, h0));
  const T rr = vfma(d, h0, gzr);
  const T two = vconst<T>(2.f);
  const T pt = vfma(two, c0, vnegz(a.template q<QP2>()));   // 2 c0 exact
  const T r0v = a.template q<QR0>();
  const T rt = vfma(two, r0v, vnegz(a.template q<QR2>()));
  p1 = vfma(sc, pp, pt);
  r1 = vfma(sc, rr, rt);
}

// ---- single-field rotated operator (the SPEC's tti_gxx_kernel):
// m u_tt = G u,  G u = sum_i D_i (a_i g),  g = sum_j a_j D_j u  (nested first
// derivatives, the reference symbolics' Deriv(a * Deriv) lowering); solved:
// u1 = 2 u0 - u2 + dt^2/m G u0.  Same operation order as the TTI routines.
template <int R, class A>
__device__ __forceinline__ typename A::T g1_point(const A& a, const TTICoef& c) {
  using T = typename A::T;
  const T ax = a.template q<QAX>(), ay = a.template q<QAY>(), az = a.template q<QAZ>();
  T g = vfma(ax, dcentral<R, 0, TP>(a, c.d1[0]), vconst<T>(0.f));
  g = vfma(ay, dcentral<R, 1, TP>(a, c.d1[1]), g);
  return vfma(az, dcentral<R, 2, TP>(a, c.d1[2]), g);
}

template <int R, class A>
__device__ __forceinline__ typename A::T rot_point(const A& a, const TTICoef& c) {
  using T = typename A::T;
  T G = outer<R, 0, TAX, TGP>(a, c.d1[0]);
  G = vadd(G, outer<R, 1, TAY, TGP>(a, c.d1[1]));
  G = vadd(G, outer<R, 2, TAZ, TGP>(a, c.d1[2]));
  const T sc = tti_scale(c, a.template q<QM>());
  const T ut = vfma(vconst<T>(2.f), a.template q<QR0>(), vnegz(a.template q<QP2>()));
  return vfma(sc, G, ut);
}

// ---- generic launch ---------------------------------------------------------

struct TTIGlobalAcc {
  using T = float;
  const float* const* tap;
  const float* const* pnt;
  int64_t i, s[3];
  template <int F, int AX>
  __device__ __forceinline__ float t(int k) const { return __ldg(tap[F] + i + k * s[AX]); }
  template <int Q>
  __device__ __forceinline__ float q() const { return __ldg(pnt[Q] + i); }
};

struct TTIGeneric {
  const float* tap[NT_];
  const float* pnt[NQ_];
  float* out[2];
  Geom g;
  TTICoef c;
};

template <int R>
__global__ void __launch_bounds__(256) tti_g(TTIGeneric p) {
  const int z = p.g.lo[2] + blockIdx.x * 32 + threadIdx.x;
  const int y = p.g.lo[1] + blockIdx.y * 8 + threadIdx.y;
  const int x = p.g.lo[0] + blockIdx.z;
  if (z >= p.g.hi[2] || y >= p.g.hi[1]) return;
  const int64_t i = x * p.g.sx + y * p.g.sy + z;
  TTIGlobalAcc a{p.tap, p.pnt, i, {p.g.sx, p.g.sy, 1}};
  float gp, gr;
  g_point<R>(a, p.c, gp, gr);
  p.out[0][i] = gp;
  p.out[1][i] = gr;
}

template <int R>
__global__ void __launch_bounds__(256) tti_update(TTIGeneric p, const Push push) {
  const int z = p.g.lo[2] + blockIdx.x * 32 + threadIdx.x;
  const int y = p.g.lo[1] + blockIdx.y * 8 + threadIdx.y;
  const int x = p.g.lo[0] + blockIdx.z;
  if (z >= p.g.hi[2] || y >= p.g.hi[1]) return;
  const int64_t i = x * p.g.sx + y * p.g.sy + z;
  TTIGlobalAcc a{p.tap, p.pnt, i, {p.g.sx, p.g.sy, 1}};
  float p1, r1;
  u_point<R>(a, p.c, p1, r1);
  p.out[0][i] = p1;
  p.out[1][i] = r1;
  if (push.ndir) {
    const float v[2] = {p1, r1};
    push_point(push, x, y, z, v, 2);
  }
}

template <int R>
__global__ void __launch_bounds__(256) rot_g(TTIGeneric p) {
  const int z = p.g.lo[2] + blockIdx.x * 32 + threadIdx.x;
  const int y = p.g.lo[1] + blockIdx.y * 8 + threadIdx.y;
  const int x = p.g.lo[0] + blockIdx.z;
  if (z >= p.g.hi[2] || y >= p.g.hi[1]) return;
  const int64_t i = x * p.g.sx + y * p.g.sy + z;
  TTIGlobalAcc a{p.tap, p.pnt, i, {p.g.sx, p.g.sy, 1}};
  p.out[0][i] = g1_point<R>(a, p.c);
}

template <int R>
__global__ void __launch_bounds__(256) rot_update(TTIGeneric p, const Push push) {
  const int z = p.g.lo[2] + blockIdx.x * 32 + threadIdx.x;
  const int y = p.g.lo[1] + blockIdx.y * 8 + threadIdx.y;
  const int x = p.g.lo[0] + blockIdx.z;
  if (z >= p.g.hi[2] || y >= p.g.hi[1]) return;
  const int64_t i = x * p.g.sx + y * p.g.sy + z;
  TTIGlobalAcc a{p.tap, p.pnt, i, {p.g.sx, p.g.sy, 1}};
  const float v = rot_point<R>(a, p.c);
  p.out[0][i] = v;
  if (push.ndir) push_point(push, x, y, z, &v, 1);
}

// ---- stream operators --------------------------------------------------------

// pass 1: fronts {p, r}; centres {p, r}; points {ax, ay, az}
template <class Ctx>
struct GAcc {
  using T = typename Ctx::T;
  const Ctx& c;
  template <int F, int AX>
  __device__ __forceinline__ T t(int k) const {
    constexpr int fi = F == TP ? 0 : 1;
    return AX == 0 ? c.xt(fi, k) : AX == 1 ? c.ct(fi, k, 0) : c.ct(fi, 0, k);
  }
  template <int Q>
  __device__ __forceinline__ T q() const { return c.pt(Q - QAX); }
};

#ifndef SDMP_GOP_CTAS
#define SDMP_GOP_CTAS 2  // r02 A/B: 2 CTAs of 8 rows per SM (61.5 -> 63.5 GPts/s)
#endif
#ifndef SDMP_GOP_V
#define SDMP_GOP_V 2
#endif
#ifndef SDMP_GOP_ROWS
#define SDMP_GOP_ROWS 1
#endif
struct GOp {
  static constexpr bool kFrontL2 = false;  // r04 A/B: front L2 hint loses here
  static constexpr int NF = 2, NC = 2, NP = 3;
  static constexpr int kCtas = SDMP_GOP_CTAS;
  static constexpr int kRows = SDMP_GOP_ROWS;
  float* out[2];
  TTICoef k;
  template <int R, class Ctx>
  __device__ __forceinline__ void point(const Ctx& c, int64_t idx, bool m0, bool m1) const {
    GAcc<Ctx> a{c};
    typename Ctx::T gp, gr;
    g_point<R>(a, k, gp, gr);
    vstore(out[0], idx, gp, m0, m1);
    vstore(out[1], idx, gr, m0, m1);
  }
};

// pass 2: fronts {ax, gp, gr, p}; centres {ay, az, gp, gr, p};
// points {p2, r0, r2, m, epsp, delp}
template <class Ctx>
struct UAcc {
  using T = typename Ctx::T;
  const Ctx& c;
  template <int F, int AX>
  __device__ __forceinline__ T t(int k) const {
    if (AX == 0) return c.xt(F == TAX ? 0 : F == TGP ? 1 : F == TGR ? 2 : 3, k);
    constexpr int ci = F == TAY ? 0 : F == TAZ ? 1 : F == TGP ? 2 : F == TGR ? 3 : 4;
    return AX == 1 ? c.ct(ci, k, 0) : c.ct(ci, 0, k);
  }
  template <int Q>
  __device__ __forceinline__ T q() const { return c.pt(Q); }
};

#ifndef SDMP_UOP_CTAS
#define SDMP_UOP_CTAS 1
#endif
#ifndef SDMP_UOP_VN
#define SDMP_UOP_VN 2
#endif
struct UOp {
  static constexpr bool kFrontL2 = false;  // r04 A/B: front L2 hint loses here
  static constexpr int NF = 4, NC = 5, NP = 6;
  static constexpr int kCtas = SDMP_UOP_CTAS;
  // a_y is tapped along y only, a_z along z only: they stage one halo
  static constexpr unsigned kCHalo = 1u | (2u << 2) | (3u << 4) | (3u << 6) | (3u << 8);
  float* out[2];
  TTICoef k;
  template <int R, class Ctx>
  __device__ __forceinline__ void point(const Ctx& c, int64_t idx, bool m0, bool m1) const {
    UAcc<Ctx> a{c};
    typename Ctx::T p1, r1;
    u_point<R>(a, k, p1, r1);
    vstore(out[0], idx, p1, m0, m1);
    vstore(out[1], idx, r1, m0, m1);
    const typename Ctx::T o[2] = {p1, r1};
    c.push_out(o, 2, m0, m1);
  }
};

// single-field rotated operator, pass 1: fronts {u}; centres {u};
// points {ax, ay, az}
template <class Ctx>
struct RGAcc {
  using T = typename Ctx::T;
  const Ctx& c;
  template <int F, int AX>
  __device__ __forceinline__ T t(int k) const {
    return AX == 0 ? c.xt(0, k) : AX == 1 ? c.ct(0, k, 0) : c.ct(0, 0, k);
  }
  template <int Q>
  __device__ __forceinline__ T q() const { return c.pt(Q - QAX); }
};

struct RGOp {
  static constexpr bool kFrontL2 = false;  // r04 A/B: front L2 hint loses here
  static constexpr int NF = 1, NC = 1, NP = 3;
  static constexpr int kStagesWide = 6;  // r04 A/B (stream.cuh StagesWideOf)
  float* out;
  TTICoef k;
  template <int R, class Ctx>
  __device__ __forceinline__ void point(const Ctx& c, int64_t idx, bool m0, bool m1) const {
    RGAcc<Ctx> a{c};
    vstore(out, idx, g1_point<R>(a, k), m0, m1);
  }
};

// pass 2: fronts {ax, g}; centres {ay, az, g}; points {u0, u2, m}
template <class Ctx>
struct RUAcc {
  using T = typename Ctx::T;
  const Ctx& c;
  template <int F, int AX>
  __device__ __forceinline__ T t(int k) const {
    if (AX == 0) return c.xt(F == TAX ? 0 : 1, k);
    constexpr int ci = F == TAY ? 0 : F == TAZ ? 1 : 2;
    return AX == 1 ? c.ct(ci, k, 0) : c.ct(ci, 0, k);
  }
  template <int Q>
  __device__ __forceinline__ T q() const { return c.pt(Q == QR0 ? 0 : Q == QP2 ? 1 : 2); }
};

struct RUOp {
  static constexpr bool kFrontL2 = false;  // r04 A/B: front L2 hint loses here
  static constexpr int NF = 2, NC = 3, NP = 3;
  static constexpr int kStagesWide = 6;  // r04 A/B (stream.cuh StagesWideOf)
  static constexpr unsigned kCHalo = 1u | (2u << 2) | (3u << 4);  // a_y: y, a_z: z, g: both
  float* out;
  TTICoef k;
  template <int R, class Ctx>
  __device__ __forceinline__ void point(const Ctx& c, int64_t idx, bool m0, bool m1) const {
    RUAcc<Ctx> a{c};
    const typename Ctx::T o = rot_point<R>(a, k);
    vstore(out, idx, o, m0, m1);
    c.push_out(&o, 1, m0, m1);
  }
};

// Launch shape per radius (rows TY, z points per thread V): packed fp32x2
// (V = 2) while the per-thread registers fit without spills (ptxas -v),
// fewer rows as R grows; scalar for the widest update stencils.
template <int R, class Op>
static int launch_tti_stream(const Op& op, const Geom& g, const int64_t full[3],
                             const float* const* arrs, cudaStream_t st,
                             const Push* push = nullptr) {
  constexpr bool upd = Op::NF == 4;
  // thin y-slabs (full-mode OWNED boxes, SO rows high): matching tile height
  const int ny = g.hi[1] - g.lo[1];
  if constexpr (R <= 2) {
    if (ny <= 4) return launch_stream_op<R, 4, 2>(op, g, full, arrs, st, push);
    return launch_stream_op<R, 16, 2>(op, g, full, arrs, st, push);
  } else if constexpr (R <= 4) {
#ifndef SDMP_GOP_TY
#define SDMP_GOP_TY 8
#endif
#ifndef SDMP_UOP_TY
#define SDMP_UOP_TY 11  // r04 A/B: 12 warps (168-register cap) beat 13 (128 cap): 67.4 vs 66.3 GPts/s
#endif
    constexpr int VG = upd ? SDMP_UOP_VN : SDMP_GOP_V;
    if (ny <= 8) return launch_stream_op<R, 8, VG>(op, g, full, arrs, st, push);
    return launch_stream_op<R, upd ? SDMP_UOP_TY : SDMP_GOP_TY, VG>(op, g, full, arrs, st, push);
  } else {
    // r02 A/B (512^3): g pass 16 rows at R = 5-6
    // r03 A/B (tools/ab_ttiw.sh, 512^3, under the x-window unroll): update
    // pass 8 rows x 2 points from R = 5 (SO-12 45.4 -> 48.2, SO-16 33.9 ->
    // 35.4), g pass 12 rows at R = 7-8 (SO-16 +2.5%)
#ifndef SDMP_TTI_GTYW
#define SDMP_TTI_GTYW 12
#endif
#ifndef SDMP_TTI_UTYW
#define SDMP_TTI_UTYW 8
#endif
#ifndef SDMP_TTI_UVW
#define SDMP_TTI_UVW 2
#endif
    // 9-warp CTAs (8 rows + producer) are register-capped at 168 per thread
    // (ptxas rounds the CTA up to 12 warps): the update pass at R >= 7
    // needs more, so it runs 7-row tiles (8 warps, 255 registers, no spills)
#ifndef SDMP_TTI_UTY7_MINR
#define SDMP_TTI_UTY7_MINR 7
#endif
    constexpr int TYU = R >= SDMP_TTI_UTY7_MINR ? 7 : SDMP_TTI_UTYW;
#ifndef SDMP_TTI_GTYM
#define SDMP_TTI_GTYM 16
#endif
    constexpr int TYW = upd ? TYU : (R <= 6 ? SDMP_TTI_GTYM : SDMP_TTI_GTYW);
    constexpr int VW = upd ? SDMP_TTI_UVW : 2;
    constexpr int TYT = upd && R >= SDMP_TTI_UTY7_MINR ? 7 : 8;
    if (ny <= 8) return launch_stream_op<R, TYT, VW>(op, g, full, arrs, st, push);
    return launch_stream_op<R, TYW, VW>(op, g, full, arrs, st, push);
  }
}

// FULL-shaped scratch pair per (device, size), grow-only, never freed
// before process exit (the plan reuses it every step).
static std::pair<float*, float*> scratch(int64_t n) {
  static std::mutex mu;
  static std::map<std::pair<int, int64_t>, std::pair<float*, float*>> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_pair(dev, n);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  float *a = nullptr, *b = nullptr;
  if (cudaMalloc(&a, n * sizeof(float)) != cudaSuccess) return {nullptr, nullptr};
  if (cudaMalloc(&b, n * sizeof(float)) != cudaSuccess) {
    cudaFree(a);
    return {nullptr, nullptr};
  }
  cudaMemset(a, 0, n * sizeof(float));
  cudaMemset(b, 0, n * sizeof(float));
  cache[key] = {a, b};
  return {a, b};
}

static int variant_env() {
  // 1 forces the generic kernels (tests compare both launch shapes bitwise)
  const char* e = getenv("SDMP_TTI_VARIANT");
  return e ? atoi(e) : 0;
}

#include "tti_fused.cuh"

// Tile rows of the single-pass rotated operator.  With one field the
// x-window and accumulators take half the TTI pair's registers, so 16-row
// tiles (16 + R + 2 consumer warps at <= 80 registers, no spills) fit; the
// g work on halo rows / columns drops from 2.25x to 1.69x at R = 4.  r04 A/B
// (512^3): SO-6 120.4 -> 163.9 GPts/s (0.52 -> 0.71), SO-8 111.9 -> 131.9
// (0.48 -> 0.57), SO-4 unchanged (profiles/round2_ab_rot_rows.txt).
#ifndef SDMP_ROT_FTY
#define SDMP_ROT_FTY 16
#endif

template <int R>
static int launch(TTIGeneric& p, cudaStream_t st, const int64_t full[3], const Push& push) {
#ifndef SDMP_TTI_FUSED_MAXR
#define SDMP_TTI_FUSED_MAXR 3
#endif
  if constexpr (R <= SDMP_TTI_FUSED_MAXR) {
    // single pass (tti_fused.cuh) where it beats the two passes (r04, 512^3,
    // unrolled, bound dt^2/m: SO-4 92.7 vs 70.1 GPts/s, SO-6 74.5 vs 68.1;
    // SO-8 49.5 vs 66.3 -- at R = 4 the 2R halo rows double the g work of
    // an 8-row tile); its
    // generic twin for boxes the TMA loads cannot cover and for the bitwise
    // tests (SDMP_TTI_VARIANT=1)
    const float* in[10] = {p.tap[TP], p.pnt[QP2], p.tap[TR], p.pnt[QR2], p.pnt[QM],
                           p.pnt[QE], p.pnt[QD], p.pnt[QAX], p.pnt[QAY], p.pnt[QAZ]};
    if (variant_env() != 1 && fused_fits<R>(p.g) && tma_ok(full, in, 10))
      return launch_fused<R, 2>(p, st, full, push);
    dim3 b(32, 8);
    dim3 g2((p.g.hi[2] - p.g.lo[2] + 31) / 32, (p.g.hi[1] - p.g.lo[1] + 7) / 8,
            p.g.hi[0] - p.g.lo[0]);
    tti_fused_generic<R><<<g2, b, 0, st>>>(p, push);
    SDMP_LAUNCHED();
    return SDMP_OK;
  }
  // SO > 8: two passes.  Pass 1 on the box grown by R (g is read up to R away by pass 2)
  TTIGeneric p1 = p;
  for (int a = 0; a < 3; ++a) {
    p1.g.lo[a] = p.g.lo[a] - R;
    p1.g.hi[a] = p.g.hi[a] + R;
  }
  p1.out[0] = const_cast<float*>(p.tap[TGP]);
  p1.out[1] = const_cast<float*>(p.tap[TGR]);
  const float* a1[7] = {p.tap[TP], p.tap[TR], p.tap[TP], p.tap[TR], p.pnt[QAX], p.pnt[QAY],
                        p.pnt[QAZ]};
  const float* a2[15] = {p.tap[TAX], p.tap[TGP], p.tap[TGR], p.tap[TP],
                         p.tap[TAY], p.tap[TAZ], p.tap[TGP], p.tap[TGR], p.tap[TP],
                         p.pnt[QP2], p.pnt[QR0], p.pnt[QR2], p.pnt[QM], p.pnt[QE], p.pnt[QD]};
  const bool stream = variant_env() != 1 && stream_fits(p1.g, R) && stream_fits(p.g, R) &&
                      tma_ok(full, a1, 7) && tma_ok(full, a2, 15);
  dim3 b(32, 8);
  if (stream) {
    GOp g{};
    g.out[0] = p1.out[0];
    g.out[1] = p1.out[1];
    g.k = p.c;
    int rc = launch_tti_stream<R>(g, p1.g, full, a1, st);
    if (rc) return rc;
    UOp u{};
    u.out[0] = p.out[0];
    u.out[1] = p.out[1];
    u.k = p.c;
    return launch_tti_stream<R>(u, p.g, full, a2, st, &push);
  }
  dim3 g1((p1.g.hi[2] - p1.g.lo[2] + 31) / 32, (p1.g.hi[1] - p1.g.lo[1] + 7) / 8,
          p1.g.hi[0] - p1.g.lo[0]);
  tti_g<R><<<g1, b, 0, st>>>(p1);
  SDMP_LAUNCHED();
  dim3 g2((p.g.hi[2] - p.g.lo[2] + 31) / 32, (p.g.hi[1] - p.g.lo[1] + 7) / 8,
          p.g.hi[0] - p.g.lo[0]);
  tti_update<R><<<g2, b, 0, st>>>(p, push);
  SDMP_LAUNCHED();
  return SDMP_OK;
}

int tti_update_entry(cudaStream_t st, const float* const in[10], float* p1, float* r1,
                     const int64_t full[3], const int64_t lo[3], const int64_t hi[3],
                     int32_t radius, const float* lap_c, const float* d1_c, float dt2,
                     const Push* push_in) {
  const int m_is_scale = (radius & SDMP_VARIANT_M_IS_SCALE) ? 1 : 0;
  radius &= 0xff;
  const Push nopush{};
  const Push& push = push_in ? *push_in : nopush;
  TTIGeneric p{};
  int rc = make_geom(full, lo, hi, &p.g);
  if (rc) return rc;
  if (box_empty(p.g)) return SDMP_OK;
  SDMP_CHECK(radius >= 1 && radius <= SDMP_MAX_RADIUS, "tti radius (SO/2) outside 1..8");
  for (int i = 0; i < 10; ++i) SDMP_CHECK(in[i] != nullptr, "tti inputs must be non-null");
  for (int a = 0; a < 3; ++a)
    SDMP_CHECK(lo[a] >= 2 * radius && hi[a] + 2 * radius <= full[a],
               "tti box + 2*radius exceeds FULL (halo must be >= SO)");
  auto sc = scratch(full[0] * full[1] * full[2]);
  if (!sc.first) {
    set_error("tti: scratch allocation failed");
    return SDMP_ECUDA;
  }
  // in = {p0, p2, r0, r2, m, epsp, delp, ax, ay, az}
  p.tap[TP] = in[0]; p.tap[TR] = in[2];
  p.tap[TAX] = in[7]; p.tap[TAY] = in[8]; p.tap[TAZ] = in[9];
  p.tap[TGP] = sc.first; p.tap[TGR] = sc.second;
  p.pnt[QP2] = in[1]; p.pnt[QR0] = in[2]; p.pnt[QR2] = in[3]; p.pnt[QM] = in[4];
  p.pnt[QE] = in[5]; p.pnt[QD] = in[6];
  p.pnt[QAX] = in[7]; p.pnt[QAY] = in[8]; p.pnt[QAZ] = in[9];
  p.out[0] = p1;
  p.out[1] = r1;
  float cs = 0.f;
  for (int a = 0; a < 3; ++a) {
    for (int k = 0; k < SDMP_NCOEF; ++k) {
      p.c.lap[a][k] = k <= radius ? lap_c[a * SDMP_NCOEF + k] : 0.f;
      p.c.d1[a][k] = (k >= 1 && k <= radius) ? d1_c[a * SDMP_NCOEF + k] : 0.f;
    }
    cs = cs + p.c.lap[a][0];
  }
  p.c.csum0 = cs;
  p.c.dt2 = dt2;
  p.c.m_is_scale = m_is_scale;
  switch (radius) {
    case 1: return launch<1>(p, st, full, push);
    case 2: return launch<2>(p, st, full, push);
    case 3: return launch<3>(p, st, full, push);
    case 4: return launch<4>(p, st, full, push);
    case 5: return launch<5>(p, st, full, push);
    case 6: return launch<6>(p, st, full, push);
    case 7: return launch<7>(p, st, full, push);
    case 8: return launch<8>(p, st, full, push);
  }
  set_error("tti: unsupported radius");
  return SDMP_EUNSUPPORTED;
}

template <int R>
static int launch_rot(TTIGeneric& p, cudaStream_t st, const int64_t full[3], const Push& push) {
#ifndef SDMP_ROT_FUSED_MAXR
#define SDMP_ROT_FUSED_MAXR 4  // r04 A/B (512^3, unrolled, bound dt^2/m): SO-4 187 vs 121, SO-6 120 vs 109, SO-8 111 vs 106 GPts/s
#endif
  if constexpr (R <= SDMP_ROT_FUSED_MAXR) {
    // single pass for the narrow stencils, as for TTI (tti_fused.cuh, NF = 1)
    const float* in[6] = {p.tap[TP], p.pnt[QP2], p.pnt[QM], p.pnt[QAX], p.pnt[QAY], p.pnt[QAZ]};
    if (variant_env() != 1 && fused_fits<R>(p.g) && tma_ok(full, in, 6))
      return launch_fused<R, 1, SDMP_ROT_FTY>(p, st, full, push);
    dim3 b(32, 8);
    dim3 g2((p.g.hi[2] - p.g.lo[2] + 31) / 32, (p.g.hi[1] - p.g.lo[1] + 7) / 8,
            p.g.hi[0] - p.g.lo[0]);
    rot_fused_generic<R><<<g2, b, 0, st>>>(p, push);
    SDMP_LAUNCHED();
    return SDMP_OK;
  }
  TTIGeneric p1 = p;
  for (int a = 0; a < 3; ++a) {
    p1.g.lo[a] = p.g.lo[a] - R;
    p1.g.hi[a] = p.g.hi[a] + R;
  }
  p1.out[0] = const_cast<float*>(p.tap[TGP]);
  const float* a1[5] = {p.tap[TP], p.tap[TP], p.pnt[QAX], p.pnt[QAY], p.pnt[QAZ]};
  const float* a2[8] = {p.tap[TAX], p.tap[TGP], p.tap[TAY], p.tap[TAZ], p.tap[TGP],
                        p.pnt[QR0], p.pnt[QP2], p.pnt[QM]};
  const bool stream = variant_env() != 1 && stream_fits(p1.g, R) && stream_fits(p.g, R) &&
                      tma_ok(full, a1, 5) && tma_ok(full, a2, 8);
  if (stream) {
    // r03 A/B (tools/ab_rot.sh, 512^3): g pass 8 rows at R = 3-4 (SO-8
    // 104.6 -> 110.9 GPts/s; SO-4 keeps 16), both passes 12 rows above R = 4
    // (SO-16 64.4 -> 76.6)
#ifndef SDMP_RG_TYN
#define SDMP_RG_TYN 8
#endif
#ifndef SDMP_RG_TYW
#define SDMP_RG_TYW 12
#endif
#ifndef SDMP_RU_TYN
#define SDMP_RU_TYN 16
#endif
#ifndef SDMP_RU_TYW
#define SDMP_RU_TYW 12
#endif
    constexpr int TYG = R <= 2 ? 16 : R <= 4 ? SDMP_RG_TYN : SDMP_RG_TYW;
    constexpr int TYU = R <= 4 ? SDMP_RU_TYN : SDMP_RU_TYW;
    constexpr int VU = 2;
    RGOp g{};
    g.out = p1.out[0];
    g.k = p.c;
    int rc = launch_stream_op<R, TYG, 2>(g, p1.g, full, a1, st);
    if (rc) return rc;
    RUOp u{};
    u.out = p.out[0];
    u.k = p.c;
    const int ny = p.g.hi[1] - p.g.lo[1];
    if (ny <= 8) return launch_stream_op<R, 8, 2>(u, p.g, full, a2, st, &push);
    return launch_stream_op<R, TYU, VU>(u, p.g, full, a2, st, &push);
  }
  dim3 b(32, 8);
  dim3 g1((p1.g.hi[2] - p1.g.lo[2] + 31) / 32, (p1.g.hi[1] - p1.g.lo[1] + 7) / 8,
          p1.g.hi[0] - p1.g.lo[0]);
  rot_g<R><<<g1, b, 0, st>>>(p1);
  SDMP_LAUNCHED();
  dim3 g2((p.g.hi[2] - p.g.lo[2] + 31) / 32, (p.g.hi[1] - p.g.lo[1] + 7) / 8,
          p.g.hi[0] - p.g.lo[0]);
  rot_update<R><<<g2, b, 0, st>>>(p, push);
  SDMP_LAUNCHED();
  return SDMP_OK;
}

int rot_update_entry(cudaStream_t st, const float* const in[6], float* u1,
                     const int64_t full[3], const int64_t lo[3], const int64_t hi[3],
                     int32_t radius, const float* d1_c, float dt2, const Push* push_in) {
  const int m_is_scale = (radius & SDMP_VARIANT_M_IS_SCALE) ? 1 : 0;
  radius &= 0xff;
  const Push nopush{};
  const Push& push = push_in ? *push_in : nopush;
  TTIGeneric p{};
  int rc = make_geom(full, lo, hi, &p.g);
  if (rc) return rc;
  if (box_empty(p.g)) return SDMP_OK;
  SDMP_CHECK(radius >= 1 && radius <= SDMP_MAX_RADIUS, "rotated radius (SO/2) outside 1..8");
  for (int i = 0; i < 6; ++i) SDMP_CHECK(in[i] != nullptr, "rotated inputs must be non-null");
  for (int a = 0; a < 3; ++a)
    SDMP_CHECK(lo[a] >= 2 * radius && hi[a] + 2 * radius <= full[a],
               "rotated box + 2*radius exceeds FULL (halo must be >= SO)");
  auto sc = scratch(full[0] * full[1] * full[2]);
  if (!sc.first) {
    set_error("rotated: scratch allocation failed");
    return SDMP_ECUDA;
  }
  // in = {u0, u2, m, ax, ay, az}
  p.tap[TP] = in[0];
  p.tap[TAX] = in[3]; p.tap[TAY] = in[4]; p.tap[TAZ] = in[5];
  p.tap[TGP] = sc.first;
  p.pnt[QR0] = in[0]; p.pnt[QP2] = in[1]; p.pnt[QM] = in[2];
  p.pnt[QAX] = in[3]; p.pnt[QAY] = in[4]; p.pnt[QAZ] = in[5];
  p.out[0] = u1;
  for (int a = 0; a < 3; ++a)
    for (int k = 0; k < SDMP_NCOEF; ++k)
      p.c.d1[a][k] = (k >= 1 && k <= radius) ? d1_c[a * SDMP_NCOEF + k] : 0.f;
  p.c.dt2 = dt2;
  p.c.m_is_scale = m_is_scale;
  switch (radius) {
    case 1: return launch_rot<1>(p, st, full, push);
    case 2: return launch_rot<2>(p, st, full, push);
    case 3: return launch_rot<3>(p, st, full, push);
    case 4: return launch_rot<4>(p, st, full, push);
    case 5: return launch_rot<5>(p, st, full, push);
    case 6: return launch_rot<6>(p, st, full, push);
    case 7: return launch_rot<7>(p, st, full, push);
    case 8: return launch_rot<8>(p, st, full, push);
  }
  set_error("rotated: unsupported radius");
  return SDMP_EUNSUPPORTED;
}

}  // namespace sdmp

extern "C" int sdmp_tti_update(void* stream, const float* const in[10], float* p1, float* r1,
                               const int64_t full[3], const int64_t lo[3], const int64_t hi[3],
                               int32_t radius, const float* lap_c, const float* d1_c, float dt2,
                               int32_t variant) {
  (void)variant;
  return sdmp::tti_update_entry((cudaStream_t)stream, in, p1, r1, full, lo, hi, radius, lap_c,
                                d1_c, dt2, nullptr);
}

extern "C" int sdmp_rot_update(void* stream, const float* const in[6], float* u1,
                               const int64_t full[3], const int64_t lo[3], const int64_t hi[3],
                               int32_t radius, const float* d1_c, float dt2) {
  return sdmp::rot_update_entry((cudaStream_t)stream, in, u1, full, lo, hi, radius, d1_c, dt2,
                                nullptr);
}
