// Single-pass TTI for R <= 4 (SO <= 8): included by tti.cu after the
// per-point helpers (TTICoef, dcentral, g_point, TTIGlobalAcc).
//
// One CTA owns a TY(y) x 64(z) tile and streams along x.  Per x-plane x' it
// evaluates g = a . grad f (f = p, r) on the tile grown by R rows (y) and
// OFF columns (z) -- the points the outer derivative taps -- and never writes
// g to HBM:
//   * the x part of the outer derivative, D_x(a_x g), is SCATTERED: the
//     thread that computes g at a tile point adds c_j (a_x g)(x') into the
//     2R+1 register accumulators of the outputs x' - j (j = -R..R);
//   * the y / z parts read the a_y g / a_z g products of plane x' from a
//     shared-memory plane (double buffered), gathered at x' itself;
//   * the Laplacian of p is formed at x' from the same x-window and taps;
// the output x = x' - R is complete after plane x' and is written with the
// pointwise operands (p2, r2, m, epsp, delp) staged for plane x.  HBM
// traffic = the 48 B/pt algorithmic count (plus halo re-reads from L2).
//
// Canonical per-point order (the generic twin below follows it exactly, so
// fused and generic launches give identical bits):
//   g_f(q)   = g_point (a_x Dx f, then a_y Dy f, then a_z Dz f; fma chain)
//   acc_f    = sum over planes x+j, j = -R..R ascending, of:
//                j != 0: fma(c_j, RN(a_x g_f)(x+j), acc)      c_j = sgn(j) w_|j| / h_x
//                j == 0: p: acc + (YZ_p - lap),  r: acc + YZ_r
//              with YZ_f = D_y(RN(a_y g_f)) + D_z(RN(a_z g_f)) (dcentral order)
//   h0 = -acc_p (= lap - Gzz p), gzr = acc_r, then the u_point update tail.
//
// Warp roles: TY tile warps (one row each, 2 z points per lane: g, the
// accumulators, the update), R halo warps (two of the 2R halo rows each: g
// only, a_y g stored), TY / 8 z-halo warps (the halo columns of 8 tile rows
// each: a_z g stored), one producer warp (TMA).  TY = 8 for the TTI pair,
// 16 for the one-field rotated operator (SDMP_ROT_FTY, tti.cu).

constexpr int kFTY = 8;   // tile rows (TTI; the rotated operator: SDMP_ROT_FTY)
constexpr int kFTZ = 64;  // tile columns (32 lanes x 2)

// NF = 2: the TTI pair (p, r); NF = 1: the single-field rotated operator
// (the SPEC's tti_gxx_kernel, u1 = 2 u0 - u2 + dt^2/m G u0)
template <int R, int NF = 2, int TY = kFTY>
struct FLayout {
  static constexpr int NPT = NF == 2 ? 5 : 2;  // p2 r2 m epsp delp | u2 m
  static constexpr int OFF = sround4(R);
  static constexpr int GY = TY + 2 * R;     // g-region rows
  static constexpr int GZ = kFTZ + 2 * OFF; // g-region columns
  static constexpr int CY = TY + 4 * R;     // centre tiles (taps of g)
  static constexpr int CZ = kFTZ + 4 * OFF;
  static constexpr int GREG = ((GY * GZ * 4) + 127) & ~127;
  static constexpr int CEN = ((CY * CZ * 4) + 127) & ~127;
  static constexpr int PTB = TY * kFTZ * 4;
  // stage: fronts p, r (g-region, plane x'+R) | centres p, r (plane x') |
  // a_x, a_y, a_z (g-region, plane x') | pointwise (tile, plane x'-R)
  static constexpr int O_FP = 0, O_FR = (NF - 1) * GREG, O_CP = NF * GREG;
  static constexpr int O_CR = NF * GREG + (NF - 1) * CEN;
  static constexpr int O_A = NF * GREG + NF * CEN;          // + q * GREG
  static constexpr int O_PT = (NF + 3) * GREG + NF * CEN;   // + q * PTB
  static constexpr int STAGE = O_PT + NPT * PTB;
  static constexpr int S = 3;
  // product plane: a_y g (per field), then a_z g (per field)
  static constexpr int PLANE = 2 * NF * GREG;
  static constexpr int BYTES = S * STAGE + 2 * PLANE + 2 * S * 8;
  static constexpr int NHW = R;                 // halo warps (2 rows each)
  static constexpr int NZW = TY / 8;           // z-halo warps (8 rows x 4 pairs each)
  static constexpr int NCW = TY + NHW + NZW;    // consumer warps
  static constexpr int THREADS = 32 * (NCW + 1);
  static constexpr uint32_t TX_FRONT = NF * GY * GZ * 4;
  static constexpr uint32_t TX_G = NF * CY * CZ * 4 + 3 * GY * GZ * 4;
  static constexpr uint32_t TX_PT = NPT * PTB;
};

struct FusedTTI {
  TTICoef c;
  float* out[2];
  Geom g;
};

// accessor of g_point / lap for one point pair from the staged tiles
template <int R, int W>
struct FAcc {
  using T = V2;
  using L = FLayout<R>;  // CZ does not depend on NF
  const V2 (&wp)[W];
  const V2 (&wr)[W];
  int b;            // window slot of plane x' - R (a constant after unrolling)
  const float* cp;  // centre p at this pair (centre row / column already applied)
  const float* cr;
  V2 ax, ay, az;
  __device__ __forceinline__ static V2 tap(const float* p, int dy, int dz) {
    const float* q = p + dy * L::CZ + dz;
    if (dz & 1) {
      const V2 lo = vload<2>(q - 1), hi = vload<2>(q + 1);
      return v2pack(v2hi(lo), v2lo(hi));
    }
    return vload<2>(q);
  }
  template <int F, int AX>
  __device__ __forceinline__ V2 t(int k) const {
    if (AX == 0) return F == TP ? wp[b + R + k] : wr[b + R + k];
    const float* b = F == TP ? cp : cr;
    return AX == 1 ? tap(b, k, 0) : tap(b, 0, k);
  }
  template <int Q>
  __device__ __forceinline__ V2 q() const { return Q == QAX ? ax : Q == QAY ? ay : az; }
};

// Laplacian of p at a point (x, y, z chains in that order, k ascending)
template <int R, class A>
__device__ __forceinline__ typename A::T lap_point(const A& a, const TTICoef& c) {
  using T = typename A::T;
  T lap = vcfma(c.csum0, a.template t<TP, 0>(0), vconst<T>(0.f));
#pragma unroll
  for (int k = 1; k <= R; ++k)
    lap = vcfma(c.lap[0][k], vadd(a.template t<TP, 0>(-k), a.template t<TP, 0>(k)), lap);
#pragma unroll
  for (int k = 1; k <= R; ++k)
    lap = vcfma(c.lap[1][k], vadd(a.template t<TP, 1>(-k), a.template t<TP, 1>(k)), lap);
#pragma unroll
  for (int k = 1; k <= R; ++k)
    lap = vcfma(c.lap[2][k], vadd(a.template t<TP, 2>(-k), a.template t<TP, 2>(k)), lap);
  return lap;
}

// update tail (u_point's): p1 = 2 p0 - p2 + dt2/m (e h0 + d gzr), r1 = ...
template <class T>
__device__ __forceinline__ void fused_finish(const TTICoef& c, T h0, T gzr, T p0, T r0, T p2,
                                             T r2, T m, T e, T d, T& p1, T& r1) {
  const T sc = tti_scale(c, m);
  const T pp = vfma(d, gzr, vmul(e, h0));
  const T rr = vfma(d, h0, gzr);
  const T two = vconst<T>(2.f);
  p1 = vfma(sc, pp, vfma(two, p0, vnegz(p2)));
  r1 = vfma(sc, rr, vfma(two, r0, vnegz(r2)));
}

// D along y (AX = 1) or z (AX = 2) of a product plane Q at a pair
template <int R, int AX>
__device__ __forceinline__ V2 dplane(const float* q, const float* w) {
  using L = FLayout<R>;
  auto tap = [&](int k) -> V2 {
    if (AX == 1) return vload<2>(q + k * L::GZ);
    if (k & 1) {
      const V2 lo = vload<2>(q + k - 1), hi = vload<2>(q + k + 1);
      return v2pack(v2hi(lo), v2lo(hi));
    }
    return vload<2>(q + k);
  };
  V2 acc = vcfma(w[1], vsub(tap(1), tap(-1)), v2bcast(0.f));
#pragma unroll
  for (int k = 2; k <= R; ++k) acc = vcfma(w[k], vsub(tap(k), tap(-k)), acc);
  return acc;
}

// ROLE 0: tile row (g, product planes, x scatter, Laplacian, outer y / z
// derivative, update); ROLE 1: two halo rows (g, a_y g); ROLE 2: the z-halo
// columns of the tile rows (g, a_z g)
template <int R, int ROLE, int NF, int TY>
__device__ __forceinline__ void fused_consumer(unsigned char* sm, unsigned char* plane,
                                               uint64_t* full_bar, uint64_t* empty_bar,
                                               const FusedTTI& P, const Push& push, int xa,
                                               int nit, int z0, int y0, int warp, int lane) {
  using L = FLayout<R, NF, TY>;
  constexpr int W = 2 * R + 1;
  constexpr int NP = ROLE == 1 ? 2 : 1;  // point pairs of this thread
  constexpr int GQ = L::GREG / 4;
  const Geom& g = P.g;
  int gr[NP], gc;
  if (ROLE == 0) {
    gr[0] = R + warp;
    gc = L::OFF + 2 * lane;
  } else if (ROLE == 1) {
    const int h = warp - TY;
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      const int idx = 2 * h + j;  // 0 .. 2R-1 over the halo rows
      gr[j] = idx < R ? idx : idx + TY;
    }
    gc = L::OFF + 2 * lane;
  } else {
    gr[0] = R + 8 * (warp - TY - L::NHW) + (lane >> 2);
    const int cpair = lane & 3;
    gc = cpair < 2 ? (L::OFF - 4 + 2 * cpair) : (L::OFF + kFTZ + 2 * (cpair - 2));
  }
  // output masks (tile role)
  const int z = z0 + 2 * lane, y = y0 + warp;
  const bool yin = ROLE == 0 && y < g.hi[1];
  const bool m0 = yin && z >= g.lo[2] && z < g.hi[2];
  const bool m1 = yin && z + 1 >= g.lo[2] && z + 1 < g.hi[2];

  // x-windows and accumulators unrolled by U planes: inside a group the
  // slots are constants (plane x'-R+k of sub-step u at slot u + k, output
  // x'-R+k at accumulator u + k); the live entries move down once per group
#ifndef SDMP_FUSED_UNROLL
#define SDMP_FUSED_UNROLL 2
#endif
  constexpr int U = SDMP_FUSED_UNROLL;
  constexpr int WB = W + U - 1;
  constexpr int NA = ROLE == 0 ? WB : 1;
  V2 wp[NP][WB], wr[NP][WB];
  V2 accp[NA], accr[NA];
#pragma unroll
  for (int k = 0; k < WB; ++k)
#pragma unroll
    for (int j = 0; j < NP; ++j) wp[j][k] = wr[j][k] = v2bcast(0.f);
#pragma unroll
  for (int k = 0; k < NA; ++k) accp[k] = accr[k] = v2bcast(0.f);
  V2 lapv = v2bcast(0.f);

  auto step = [&](const int i, const int u) {
    const int s = i % L::S;
    mbar_wait(&full_bar[s], (i / L::S) & 1);
    const unsigned char* st = sm + s * L::STAGE;
    float* pl = reinterpret_cast<float*>(plane + (i & 1) * L::PLANE);
    // (a) x-windows: plane x'+R lands in slot u + 2R
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      const int o = gr[j] * L::GZ + gc;
      wp[j][u + W - 1] = vload<2>(reinterpret_cast<const float*>(st + L::O_FP) + o);
      if (NF == 2) wr[j][u + W - 1] = vload<2>(reinterpret_cast<const float*>(st + L::O_FR) + o);
    }
    const bool gpl = i >= 2 * R;
    // (b) g at this thread's points, product planes, x scatter, Laplacian
    if (gpl) {
#pragma unroll
      for (int j = 0; j < NP; ++j) {
        const int o = gr[j] * L::GZ + gc;
        const int oc = (gr[j] + R) * L::CZ + gc + L::OFF;
        const float* A = reinterpret_cast<const float*>(st + L::O_A);
        FAcc<R, WB> a{wp[j], NF == 2 ? wr[j] : wp[j], u,
                      reinterpret_cast<const float*>(st + L::O_CP) + oc,
                      reinterpret_cast<const float*>(st + L::O_CR) + oc, vload<2>(A + o),
                      vload<2>(A + GQ + o), vload<2>(A + 2 * GQ + o)};
        V2 gp, grv = v2bcast(0.f);
        if constexpr (NF == 2)
          g_point<R>(a, P.c, gp, grv);
        else
          gp = g1_point<R>(a, P.c);
        // the Laplacian taps of p are g's taps: form it before the product
        // stores so the shared-memory loads are reused, not repeated (r04 A/B:
        // TTI SO-4 +3%, SO-6 +5%; profiles/round2_ab_fused_lapfirst.txt)
        if constexpr (ROLE == 0 && NF == 2) lapv = lap_point<R>(a, P.c);
        if (ROLE != 2) {  // a_y g: tapped along y (tile and halo rows)
          *reinterpret_cast<uint64_t*>(pl + o) = vmul(a.ay, gp).r;
          if (NF == 2) *reinterpret_cast<uint64_t*>(pl + GQ + o) = vmul(a.ay, grv).r;
        }
        if (ROLE != 1) {  // a_z g: tapped along z (tile rows and z-halo columns)
          *reinterpret_cast<uint64_t*>(pl + NF * GQ + o) = vmul(a.az, gp).r;
          if (NF == 2) *reinterpret_cast<uint64_t*>(pl + 3 * GQ + o) = vmul(a.az, grv).r;
        }
        if constexpr (ROLE == 0) {
          const V2 axp = vmul(a.ax, gp), axr = vmul(a.ax, grv);
          // accumulator u + k holds output x' - R + k: plane x' is its x + (R - k)
#pragma unroll
          for (int k = 0; k < W; ++k) {
            if (k == R) continue;
            const int jj = R - k;
            const float cj = jj > 0 ? P.c.d1[0][jj] : -P.c.d1[0][-jj];
            accp[u + k] = vcfma(cj, axp, accp[u + k]);
            if (NF == 2) accr[u + k] = vcfma(cj, axr, accr[u + k]);
          }
        }
      }
    }
    // (c) the product plane is complete
    named_sync(1, L::NCW * 32);
    if constexpr (ROLE == 0) {
      if (gpl) {
        // (d) y / z parts of the outer derivative at x', folded at j = 0
        const float* q = pl + gr[0] * L::GZ + gc;
        const V2 yzp = vadd(dplane<R, 1>(q, P.c.d1[1]), dplane<R, 2>(q + NF * GQ, P.c.d1[2]));
        if constexpr (NF == 2) {
          const V2 yzr = vadd(dplane<R, 1>(q + GQ, P.c.d1[1]),
                              dplane<R, 2>(q + 3 * GQ, P.c.d1[2]));
          accp[u + R] = vadd(accp[u + R], vsub(yzp, lapv));
          accr[u + R] = vadd(accr[u + R], yzr);
        } else {
          accp[u + R] = vadd(accp[u + R], yzp);
        }
        // (e) output x' - R is complete
        if (i >= 4 * R && (m0 || m1)) {
          const int x = xa - 4 * R + i;
          const float* pt = reinterpret_cast<const float*>(st + L::O_PT) + warp * kFTZ + 2 * lane;
          constexpr int PQ = L::PTB / 4;
          const int64_t idx = (int64_t)x * g.sx + (int64_t)y * g.sy + z;
          if constexpr (NF == 2) {
            V2 p1, r1;
            fused_finish(P.c, vneg(accp[u]), accr[u], wp[0][u], wr[0][u], vload<2>(pt),
                         vload<2>(pt + PQ), vload<2>(pt + 2 * PQ), vload<2>(pt + 3 * PQ),
                         vload<2>(pt + 4 * PQ), p1, r1);
            vstore(P.out[0], idx, p1, m0, m1);
            vstore(P.out[1], idx, r1, m0, m1);
            if (push.ndir) {
              const V2 o2[2] = {p1, r1};
              push_vals(push, x, y, z, o2, 2, m0, m1);
            }
          } else {
            // rot_point's tail: u1 = 2 u0 - u2 + dt^2/m G
            const V2 ut = vfma(v2bcast(2.f), wp[0][u], vnegz(vload<2>(pt)));
            const V2 u1 = vfma(tti_scale(P.c, vload<2>(pt + PQ)), accp[u], ut);
            vstore(P.out[0], idx, u1, m0, m1);
            if (push.ndir) push_vals(push, x, y, z, &u1, 1, m0, m1);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[s]);
  };

  for (int i0 = 0; i0 < nit; i0 += U) {
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i0 + u < nit) step(i0 + u, u);
    // the W-1 newest planes / the pending outputs move down one group
#pragma unroll
    for (int k = 0; k < W - 1; ++k)
#pragma unroll
      for (int j = 0; j < NP; ++j) {
        wp[j][k] = wp[j][k + U];
        if (NF == 2) wr[j][k] = wr[j][k + U];
      }
    if constexpr (ROLE == 0) {
#pragma unroll
      for (int k = 0; k < W - 1; ++k) {
        accp[k] = accp[k + U];
        if (NF == 2) accr[k] = accr[k + U];
      }
#pragma unroll
      for (int k = W - 1; k < WB; ++k) accp[k] = accr[k] = v2bcast(0.f);
    }
  }
}

template <int R, int NF, int TY>
__global__ void __launch_bounds__(FLayout<R, NF, TY>::THREADS, 1)
tti_fused(const __grid_constant__ TMaps maps, const FusedTTI P, const int xchunk,
          const __grid_constant__ Push push) {
  using L = FLayout<R, NF, TY>;
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = smraw;
  unsigned char* plane = sm + L::S * L::STAGE;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(plane + 2 * L::PLANE);
  uint64_t* empty_bar = full_bar + L::S;
  const int lane = threadIdx.x, warp = threadIdx.y;
  const Geom& g = P.g;
  if (lane == 0 && warp == 0) {
    for (int s = 0; s < L::S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], L::NCW);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int z0 = (g.lo[2] & ~3) + blockIdx.x * kFTZ;
  const int y0 = g.lo[1] + blockIdx.y * TY;
  const int xa = g.lo[0] + blockIdx.z * xchunk;
  const int xb = min(xa + xchunk, g.hi[0]);
  const int nit = (xb - xa) + 4 * R;

  if (warp == L::NCW) {  // producer
    if (lane == 0) {
      for (int i = 0; i < nit; ++i) {
        const int s = i % L::S;
        mbar_wait(&empty_bar[s], ((i / L::S) & 1) ^ 1);
        unsigned char* st = sm + s * L::STAGE;
        const int xf = xa - 2 * R + i;  // front plane; g plane xf - R; output plane xf - 2R
        const bool gpl = i >= 2 * R, upl = i >= 4 * R;
        mbar_arrive_expect_tx(&full_bar[s], L::TX_FRONT + (gpl ? L::TX_G : 0u) +
                                                (upl ? L::TX_PT : 0u));
        // maps: fronts [0, NF), centres [NF, 2NF), a [2NF, 2NF+3), points after
#pragma unroll
        for (int f = 0; f < NF; ++f)
          tma_load_3d(st + L::O_FP + f * L::GREG, &maps.m[f], &full_bar[s], z0 - L::OFF, y0 - R,
                      xf);
        if (gpl) {
#pragma unroll
          for (int f = 0; f < NF; ++f)
            tma_load_3d(st + L::O_CP + f * L::CEN, &maps.m[NF + f], &full_bar[s],
                        z0 - 2 * L::OFF, y0 - 2 * R, xf - R);
#pragma unroll
          for (int q = 0; q < 3; ++q)
            tma_load_3d(st + L::O_A + q * L::GREG, &maps.m[2 * NF + q], &full_bar[s],
                        z0 - L::OFF, y0 - R, xf - R);
        }
        if (upl) {
#pragma unroll
          for (int q = 0; q < L::NPT; ++q)
            tma_load_3d(st + L::O_PT + q * L::PTB, &maps.m[2 * NF + 3 + q], &full_bar[s], z0,
                        y0, xf - 2 * R);
        }
      }
    }
    return;
  }
  // consumers: one loop per role (separate register allocations)
  if (warp < TY)
    fused_consumer<R, 0, NF, TY>(sm, plane, full_bar, empty_bar, P, push, xa, nit, z0, y0, warp,
                             lane);
  else if (warp < TY + L::NHW)
    fused_consumer<R, 1, NF, TY>(sm, plane, full_bar, empty_bar, P, push, xa, nit, z0, y0, warp,
                             lane);
  else
    fused_consumer<R, 2, NF, TY>(sm, plane, full_bar, empty_bar, P, push, xa, nit, z0, y0, warp,
                             lane);
}

// ---- generic twin: one thread per output point, same order ------------------

template <int R>
__device__ __forceinline__ void g_at(const TTIGeneric& p, int64_t i, float& gp, float& gr) {
  TTIGlobalAcc a{p.tap, p.pnt, i, {p.g.sx, p.g.sy, 1}};
  g_point<R>(a, p.c, gp, gr);
}

template <int R>
__global__ void __launch_bounds__(256) tti_fused_generic(TTIGeneric p, const Push push) {
  const int z = p.g.lo[2] + blockIdx.x * 32 + threadIdx.x;
  const int y = p.g.lo[1] + blockIdx.y * 8 + threadIdx.y;
  const int x = p.g.lo[0] + blockIdx.z;
  if (z >= p.g.hi[2] || y >= p.g.hi[1]) return;
  const int64_t sx = p.g.sx, sy = p.g.sy;
  const int64_t i = x * sx + y * sy + z;
  TTIGlobalAcc a{p.tap, p.pnt, i, {sx, sy, 1}};
  const float lap = lap_point<R>(a, p.c);
  auto qprod = [&](int64_t j, int q, float& vp, float& vr) {  // RN(a_q g) at index j
    float gp, gr;
    g_at<R>(p, j, gp, gr);
    const float aq = __ldg(p.pnt[QAX + q] + j);
    vp = __fmul_rn(aq, gp);
    vr = __fmul_rn(aq, gr);
  };
  float accp = 0.f, accr = 0.f;
#pragma unroll 1
  for (int jj = -R; jj <= R; ++jj) {
    if (jj == 0) {
      float dyp = 0.f, dyr = 0.f, dzp = 0.f, dzr = 0.f;
#pragma unroll 1
      for (int k = 1; k <= R; ++k) {
        float pp, pr, mp, mr;
        qprod(i + k * sy, 1, pp, pr);
        qprod(i - k * sy, 1, mp, mr);
        dyp = __fmaf_rn(p.c.d1[1][k], __fsub_rn(pp, mp), dyp);
        dyr = __fmaf_rn(p.c.d1[1][k], __fsub_rn(pr, mr), dyr);
        qprod(i + k, 2, pp, pr);
        qprod(i - k, 2, mp, mr);
        dzp = __fmaf_rn(p.c.d1[2][k], __fsub_rn(pp, mp), dzp);
        dzr = __fmaf_rn(p.c.d1[2][k], __fsub_rn(pr, mr), dzr);
      }
      accp = __fadd_rn(accp, __fsub_rn(__fadd_rn(dyp, dzp), lap));
      accr = __fadd_rn(accr, __fadd_rn(dyr, dzr));
    } else {
      float vp, vr;
      qprod(i + jj * sx, 0, vp, vr);
      const float cj = jj > 0 ? p.c.d1[0][jj] : -p.c.d1[0][-jj];
      accp = __fmaf_rn(cj, vp, accp);
      accr = __fmaf_rn(cj, vr, accr);
    }
  }
  float p1, r1;
  fused_finish<float>(p.c, -accp, accr, __ldg(p.tap[TP] + i), __ldg(p.pnt[QR0] + i),
                      __ldg(p.pnt[QP2] + i), __ldg(p.pnt[QR2] + i), __ldg(p.pnt[QM] + i),
                      __ldg(p.pnt[QE] + i), __ldg(p.pnt[QD] + i), p1, r1);
  p.out[0][i] = p1;
  p.out[1][i] = r1;
  if (push.ndir) {
    const float v[2] = {p1, r1};
    push_point(push, x, y, z, v, 2);
  }
}

// single-field twin (rotated operator): same order with one accumulator, no
// Laplacian, rot_point's update tail
template <int R>
__global__ void __launch_bounds__(256) rot_fused_generic(TTIGeneric p, const Push push) {
  const int z = p.g.lo[2] + blockIdx.x * 32 + threadIdx.x;
  const int y = p.g.lo[1] + blockIdx.y * 8 + threadIdx.y;
  const int x = p.g.lo[0] + blockIdx.z;
  if (z >= p.g.hi[2] || y >= p.g.hi[1]) return;
  const int64_t sx = p.g.sx, sy = p.g.sy;
  const int64_t i = x * sx + y * sy + z;
  auto qprod = [&](int64_t j, int q) {  // RN(a_q g) at index j
    TTIGlobalAcc a{p.tap, p.pnt, j, {sx, sy, 1}};
    return __fmul_rn(__ldg(p.pnt[QAX + q] + j), g1_point<R>(a, p.c));
  };
  float acc = 0.f;
#pragma unroll 1
  for (int jj = -R; jj <= R; ++jj) {
    if (jj == 0) {
      float dy = 0.f, dz = 0.f;
#pragma unroll 1
      for (int k = 1; k <= R; ++k) {
        dy = __fmaf_rn(p.c.d1[1][k], __fsub_rn(qprod(i + k * sy, 1), qprod(i - k * sy, 1)), dy);
        dz = __fmaf_rn(p.c.d1[2][k], __fsub_rn(qprod(i + k, 2), qprod(i - k, 2)), dz);
      }
      acc = __fadd_rn(acc, __fadd_rn(dy, dz));
    } else {
      const float cj = jj > 0 ? p.c.d1[0][jj] : -p.c.d1[0][-jj];
      acc = __fmaf_rn(cj, qprod(i + jj * sx, 0), acc);
    }
  }
  const float ut = __fmaf_rn(2.f, __ldg(p.pnt[QR0] + i), __fsub_rn(0.f, __ldg(p.pnt[QP2] + i)));
  const float v = __fmaf_rn(tti_scale(p.c, __ldg(p.pnt[QM] + i)), acc, ut);
  p.out[0][i] = v;
  if (push.ndir) push_point(push, x, y, z, &v, 1);
}

// host: fused launch.  NF = 2 (TTI): maps {p, r | p, r | ax, ay, az | p2, r2,
// m, epsp, delp}; NF = 1 (rotated): {u0 | u0 | ax, ay, az | u2, m}
template <int R, int NF, int TY = kFTY>
static int launch_fused(const TTIGeneric& p, cudaStream_t st, const int64_t full[3],
                        const Push& push) {
  using L = FLayout<R, NF, TY>;
  static int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    SDMP_CUDA(cudaFuncSetAttribute(tti_fused<R, NF, TY>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, L::BYTES));
    attr_dev = dev;
  }
  TMaps maps;
  const float* src2[12] = {p.tap[TP], p.tap[TR], p.tap[TP], p.tap[TR], p.pnt[QAX], p.pnt[QAY],
                           p.pnt[QAZ], p.pnt[QP2], p.pnt[QR2], p.pnt[QM], p.pnt[QE], p.pnt[QD]};
  const float* src1[7] = {p.tap[TP], p.tap[TP], p.pnt[QAX], p.pnt[QAY], p.pnt[QAZ],
                          p.pnt[QP2], p.pnt[QM]};
  const float* const* src = NF == 2 ? src2 : src1;
  constexpr int NMAP = 2 * NF + 3 + L::NPT;
  for (int k = 0; k < NMAP; ++k) {
    const bool front = k < NF, cen = k >= NF && k < 2 * NF, am = k >= 2 * NF && k < 2 * NF + 3;
    const int bz = front || am ? L::GZ : cen ? L::CZ : kFTZ;
    const int by = front || am ? L::GY : cen ? L::CY : TY;
    int rc = make_tmap_3d(&maps.m[k], src[k], full, bz, by, k >= 2 * NF + 3);
    if (rc) return rc;
  }
  FusedTTI f{};
  f.c = p.c;
  f.out[0] = p.out[0];
  f.out[1] = p.out[1];
  f.g = p.g;
  const int nz = p.g.hi[2] - p.g.lo[2], ny = p.g.hi[1] - p.g.lo[1], nx = p.g.hi[0] - p.g.lo[0];
  const int tz = (nz + (p.g.lo[2] & 3) + kFTZ - 1) / kFTZ, ty = (ny + TY - 1) / TY;
  int nch = stream_chunks((int64_t)tz * ty, nx, 2 * R, 1);
  const int chunk = (nx + nch - 1) / nch;
  nch = (nx + chunk - 1) / chunk;
  SDMP_CHECK(nch <= 65535 && ty <= 65535, "grid too large");
  dim3 grid(tz, ty, nch), block(32, L::NCW + 1);
  tti_fused<R, NF, TY><<<grid, block, L::BYTES, st>>>(maps, f, chunk, push);
  SDMP_LAUNCHED();
  return SDMP_OK;
}

// loads of the fused kernel start at (z0 - 2 OFF, y0 - 2R, x0 - 2R)
template <int R>
inline bool fused_fits(const Geom& g) {
  return (g.lo[2] & ~3) - 2 * FLayout<R>::OFF >= 0 && g.lo[1] - 2 * R >= 0 &&
         g.lo[0] - 2 * R >= 0;
}
