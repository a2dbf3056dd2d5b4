// Generic TMA streaming engine for multi-field stencils on sm_100a.
//
// A CTA owns a (32*V)(z) x TY(y) tile and streams along x.  One producer
// warp fills an S-stage shared-memory ring with cp.async.bulk.tensor 3D tile
// loads (mbarrier complete_tx); TY consumer warps compute V consecutive z
// points per thread (V = 2: packed fp32x2 arithmetic, 64-bit LDS/STG).
// Per pipeline iteration i (plane xa-R+i):
//
//   NF "front" tiles  [TY][32V]              -> per-field x-window registers
//   NC "centre" tiles [TY+2R][32V+2*OFF]     -> y / z taps (TMA zero-fills OOB;
//                                               an op can drop the y or z halo
//                                               of a tile tapped along one axis)
//   NP "point" tiles  [TY][32V]              -> pointwise operands
//
// front tiles run 2R planes ahead of the centre/point tiles, so at
// iteration i >= 2R the consumer holds planes x-R..x+R of every front field
// in registers and the centre/point tiles of plane x in the stage.
//
// The operator `Op` supplies
//   static constexpr int NF, NC, NP;
//   template <int R, class Ctx> __device__ void point(const Ctx&, int64_t idx,
//                                                      bool m0, bool m1) const;
// and the per-point arithmetic is shared with the one-thread-per-point
// generic kernels through accessor / value-type templates (vmath.cuh), so
// both launch shapes give identical bits.
#pragma once

#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "tma.cuh"
#include "vmath.cuh"

namespace sdmp {

constexpr int kSZ = 32;  // lanes along z

__host__ __device__ constexpr int sround4(int r) { return (r + 3) & ~3; }

// Centre-tile halo mask: 2 bits per centre tile c (bit 2c: the tile carries
// the R-row y halo, bit 2c+1: the OFF-column z halo).  An op whose tile is
// only tapped along one axis stages just that halo (Op::kCHalo; default all
// tiles carry both).
#ifndef SDMP_STREAM_STAGES
#define SDMP_STREAM_STAGES 4
#endif
// Front tiles are loaded with an L2 evict_last hint (their rows come back R
// planes later as centre-tile interiors and neighbours' y halos) unless the
// op sets kFrontL2 = false.  r04 A/B (profiles/round2_ab_front_l2.txt):
// visco SO-16 +4.5%, elastic SO-16 +1.8%, SO-8 +1%, damped SO-16 +0.8%;
// the TTI / rotated passes lose up to 2% and opt out.
#ifndef SDMP_STREAM_FRONT_L2
#define SDMP_STREAM_FRONT_L2 1
#endif
constexpr unsigned kHaloYZ = 0xFFFFFFFFu;
__host__ __device__ constexpr bool halo_y(unsigned m, int c) { return (m >> (2 * c)) & 1u; }
__host__ __device__ constexpr bool halo_z(unsigned m, int c) { return (m >> (2 * c + 1)) & 1u; }

template <int R, int TY, int V, int NF, int NC, int NP, int CT = 1, unsigned M = kHaloYZ,
          int RB = 1, int SMAX = SDMP_STREAM_STAGES>
struct SLayout {
  static constexpr int TZ = kSZ * V;
  static constexpr int OFF = sround4(R);
  static constexpr int FRONT = TZ * TY * 4;
  // centre tile c: rows (y halo R each side if masked in), columns (z halo OFF)
  static constexpr int cy(int c) { return TY + (halo_y(M, c) ? 2 * R : 0); }
  static constexpr int cz(int c) { return TZ + (halo_z(M, c) ? 2 * OFF : 0); }
  static constexpr int cbytes(int c) { return ((cz(c) * cy(c) * 4) + 127) & ~127; }
  static constexpr int coff(int c) {
    int o = 0;
    for (int i = 0; i < c; ++i) o += cbytes(i);
    return o;
  }
  static constexpr int ctx_bytes() {
    int b = 0;
    for (int i = 0; i < NC; ++i) b += cz(i) * cy(i) * 4;
    return b;
  }
  static constexpr int CENTERS = coff(NC);
  static constexpr int STAGE = NF * FRONT + CENTERS + NP * FRONT;
  static constexpr int S0 = (220 * 1024) / CT / STAGE;  // CT resident CTAs per SM
  static constexpr int S = S0 > SMAX ? SMAX : (S0 < 2 ? 2 : S0);
  static constexpr int BYTES = S * STAGE + 2 * S * 8;
  static constexpr int THREADS = 32 * (TY / RB + 1);  // consumer warps + producer
  static constexpr uint32_t TX_FRONT = NF * FRONT;
  static constexpr uint32_t TX_MAIN = NF * FRONT + ctx_bytes() + NP * FRONT;
};

constexpr int kMaxMaps = 24;
struct TMaps {
  CUtensorMap m[kMaxMaps];
};

// (r02 A/B, dropped: a register-ring x-window unrolled by 2R+1 — i-cache
// bound for the large ops; pointwise operands loaded straight from global
// memory one plane ahead instead of TMA-staged — latency bound, 1.3-1.6x
// slower stress phases.)

// Op::kRows (optional, default 1): y rows per consumer thread.  With 2 the
// two rows' point() calls sit in one block, so the y taps they share (row
// y+1's tap at dy is row y's at dy+1) are loaded from shared memory once.
template <class Op, class = void>
struct RowsOf {
  static constexpr int value = 1;
};
template <class Op>
struct RowsOf<Op, std::void_t<decltype(Op::kRows)>> {
  static constexpr int value = Op::kRows;
};

// Op::kCtas (optional, default 1): resident CTAs per SM (launch bounds and
// the shared-memory ring are sized for it)
template <class Op, class = void>
struct CtasOf {
  static constexpr int value = 1;
};
template <class Op>
struct CtasOf<Op, std::void_t<decltype(Op::kCtas)>> {
  static constexpr int value = Op::kCtas;
};

// resident CTAs per SM for a launch shape: Op::kCtas only for small tiles
// (at most 9 warps), so taller tiles keep their full register budget
template <class Op, int TY>
constexpr int ctas_for() {
  return TY / RowsOf<Op>::value + 1 <= 9 ? CtasOf<Op>::value : 1;
}

// x-window unroll (stream_kernel): U = 2 planes per group where it was
// measured faster (r03 A/B: TTI, elastic SO-16, visco SO-16, damped +1-7%),
// 1 for ops that declare Op::kUnrollMinR above R (visco stress at SO-8 lost
// 15% to register pressure).  SDMP_STREAM_UNROLL overrides (development).
#ifndef SDMP_STREAM_UNROLL
#define SDMP_STREAM_UNROLL 0
#endif
template <class Op, class = void>
struct UnrollMinR {
  static constexpr int value = 0;
};
template <class Op>
struct UnrollMinR<Op, std::void_t<decltype(Op::kUnrollMinR)>> {
  static constexpr int value = Op::kUnrollMinR;
};
template <class Op, int R>
constexpr int unroll_for() {
  return SDMP_STREAM_UNROLL ? SDMP_STREAM_UNROLL : (R >= UnrollMinR<Op>::value ? 2 : 1);
}

// Op::kStagesWide (optional): pipeline depth cap for R >= 5 (default 4).
// r04 A/B: 6 stages help the wide visco stress (+4-5%), rotated (+7%) and
// staggered velocity (+2%) ops and cost the others (damped SO-16 -12%).
template <class Op, class = void>
struct StagesWideOf {
  static constexpr int value = SDMP_STREAM_STAGES;
};
template <class Op>
struct StagesWideOf<Op, std::void_t<decltype(Op::kStagesWide)>> {
  static constexpr int value = Op::kStagesWide;
};
template <class Op, int R>
constexpr int stages_for() {
  return R >= 5 ? StagesWideOf<Op>::value : SDMP_STREAM_STAGES;
}

template <class Op, class = void>
struct FrontL2Of {
  static constexpr bool value = SDMP_STREAM_FRONT_L2 != 0;
};
template <class Op>
struct FrontL2Of<Op, std::void_t<decltype(Op::kFrontL2)>> {
  static constexpr bool value = SDMP_STREAM_FRONT_L2 != 0 && Op::kFrontL2;
};

template <class Op, class = void>
struct CHaloOf {
  static constexpr unsigned value = kHaloYZ;
};
template <class Op>
struct CHaloOf<Op, std::void_t<decltype(Op::kCHalo)>> {
  static constexpr unsigned value = Op::kCHalo;
};

template <int V> struct VType;
template <> struct VType<1> { using T = float; };
template <> struct VType<2> { using T = V2; };

template <int V>
__device__ __forceinline__ typename VType<V>::T vload(const float* p);
template <>
__device__ __forceinline__ float vload<1>(const float* p) { return *p; }
template <>
__device__ __forceinline__ V2 vload<2>(const float* p) {
  V2 o;
  o.r = *reinterpret_cast<const uint64_t*>(p);
  return o;
}

// Consumer-side view of one thread's V points.
template <int R, int TY, int V, int NF, int NC, int NP, int U = 1, unsigned M = kHaloYZ>
struct StreamCtx {
  using L = SLayout<R, TY, V, NF, NC, NP, 1, M>;
  using T = typename VType<V>::T;
  static constexpr int W = 2 * R + 1;
  static constexpr int WB = W + U - 1;
  const T (*w)[WB];  // x-windows (registers, see stream_kernel)
  const unsigned char* stage;
  int warp, lane;
  int base;          // window slot of plane x - R (a constant after unrolling)
  const Push* push;  // fused halo push (full mode OWNED slabs), ndir 0 = none
  int x, y, z;       // FULL coordinates of the thread's first point
  // plane x + k of front field f
  __device__ __forceinline__ T xt(int f, int k) const { return w[f][base + R + k]; }
  __device__ __forceinline__ const float* crow(int c, int dy) const {
    const float* base = reinterpret_cast<const float*>(stage + NF * L::FRONT + L::coff(c));
    return base + (warp + (halo_y(M, c) ? R : 0) + dy) * L::cz(c) + (halo_z(M, c) ? L::OFF : 0) +
           V * lane;
  }
  // centre tile c at (y + dy, z + dz)
  __device__ __forceinline__ T ct(int c, int dy, int dz) const {
    const float* p = crow(c, dy) + dz;
    if constexpr (V == 2) {
      // odd shift: two aligned 64-bit loads (r02 A/B: faster than two 32-bit)
      if (dz & 1) {
        const V2 lo = vload<2>(p - 1), hi = vload<2>(p + 1);
        return v2pack(v2hi(lo), v2lo(hi));
      }
    }
    return vload<V>(p);
  }
  // store n outputs of this thread's points into every neighbour HALO whose
  // receive box contains them (peer pointers over NVLink)
  __device__ __forceinline__ void push_out(const T* v, int n, bool m0, bool m1) const {
    if (push->ndir) push_vals(*push, x, y, z, v, n, m0, m1);
  }
  __device__ __forceinline__ T pt(int q) const {
    const float* base = reinterpret_cast<const float*>(stage + NF * L::FRONT + L::CENTERS +
                                                       q * L::FRONT);
    return vload<V>(base + warp * L::TZ + V * lane);
  }
};

// fused push of one thread's points (float: one point; V2: z, z + 1)
__device__ __forceinline__ void push_vals(const Push& P, int x, int y, int z, const float* v,
                                          int n, bool m0, bool) {
  if (m0) push_point(P, x, y, z, v, n);
}
__device__ __forceinline__ void push_vals(const Push& P, int x, int y, int z, const V2* v, int n,
                                          bool m0, bool m1) {
  for (int d = 0; d < P.ndir; ++d) {
    const PushGeo& g = P.geo[d];
    if (x < g.lo[0] || x >= g.hi[0] || y < g.lo[1] || y >= g.hi[1]) continue;
    const bool in0 = m0 && z >= g.lo[2] && z < g.hi[2];
    const bool in1 = m1 && z + 1 >= g.lo[2] && z + 1 < g.hi[2];
    if (!in0 && !in1) continue;
    const int64_t j = (int64_t)(x + g.off[0]) * g.psx + (int64_t)(y + g.off[1]) * g.psy +
                      (z + g.off[2]);
    for (int q = 0; q < n && q < P.nout; ++q) {
      if (!P.base[q][d]) continue;  // not read across this face
      float* dst = P.base[q][d] + j;
      if (in0 && in1 && (reinterpret_cast<uintptr_t>(dst) & 7) == 0) {
        *reinterpret_cast<uint64_t*>(dst) = v[q].r;
      } else {
        if (in0) dst[0] = v2lo(v[q]);
        if (in1) dst[1] = v2hi(v[q]);
      }
    }
  }
}

// masked store of V consecutive values at idx (m0: first point, m1: second)
// (r03 A/B: evict-first st.global.cs stores gave nothing here)
__device__ __forceinline__ void vstore(float* p, int64_t idx, float v, bool m0, bool) {
  if (m0) p[idx] = v;
}
__device__ __forceinline__ void vstore(float* p, int64_t idx, V2 v, bool m0, bool m1) {
  if (m0 && m1) {
    *reinterpret_cast<uint64_t*>(p + idx) = v.r;
  } else {
    if (m0) p[idx] = v2lo(v);
    if (m1) p[idx + 1] = v2hi(v);
  }
}

template <int R, int TY, int V, class Op>
__global__ void __launch_bounds__(
    SLayout<R, TY, V, Op::NF, Op::NC, Op::NP, 1, kHaloYZ, RowsOf<Op>::value>::THREADS,
    (ctas_for<Op, TY>()))
stream_kernel(const __grid_constant__ TMaps maps, const Op op, const Geom g, const int xchunk,
              const __grid_constant__ Push push) {
  constexpr int NF = Op::NF, NC = Op::NC, NP = Op::NP;
  constexpr unsigned M = CHaloOf<Op>::value;
  constexpr int RB = RowsOf<Op>::value;
  constexpr int NCW = TY / RB;  // consumer warps
  static_assert(TY % RB == 0, "tile rows must be a multiple of the rows per thread");
  using L = SLayout<R, TY, V, NF, NC, NP, ctas_for<Op, TY>(), M, RB, stages_for<Op, R>()>;
  using T = typename VType<V>::T;
  // __align__(1024) keeps TMA destinations aligned without integer pointer
  // arithmetic, so the consumers keep shared-space pointers (LDS)
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = smraw;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(sm + L::S * L::STAGE);
  uint64_t* empty_bar = full_bar + L::S;
  const int lane = threadIdx.x, warp = threadIdx.y;
  if (lane == 0 && warp == 0) {
    for (int s = 0; s < L::S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], NCW);
    }
    fence_barrier_init();
  }
  __syncthreads();
  // TMA boxes must start on a 16 B boundary along z: tiles are aligned down
  // to a multiple of 4 floats and lanes outside the box are masked off.
  const int z0 = (g.lo[2] & ~3) + blockIdx.x * L::TZ;
  const int y0 = g.lo[1] + blockIdx.y * TY;
  const int xa = g.lo[0] + blockIdx.z * xchunk;
  const int xb = min(xa + xchunk, g.hi[0]);
  const int nit = (xb - xa) + 2 * R;

  if (warp == NCW) {  // producer
    if (lane == 0) {
      for (int i = 0; i < nit; ++i) {
        const int s = i % L::S;
        mbar_wait(&empty_bar[s], ((i / L::S) & 1) ^ 1);
        unsigned char* st = sm + s * L::STAGE;
        const bool main = i >= 2 * R;
        mbar_arrive_expect_tx(&full_bar[s], main ? L::TX_MAIN : L::TX_FRONT);
        const int xf = xa - R + i;
#pragma unroll
        for (int f = 0; f < NF; ++f) {
          if constexpr (FrontL2Of<Op>::value)
            tma_load_3d_hint(st + f * L::FRONT, &maps.m[f], &full_bar[s], z0, y0, xf,
                             l2_policy_evict_last());
          else
            tma_load_3d(st + f * L::FRONT, &maps.m[f], &full_bar[s], z0, y0, xf);
        }
        if (main) {
          const int x = xa + i - 2 * R;
#pragma unroll
          for (int c = 0; c < NC; ++c)
            tma_load_3d(st + NF * L::FRONT + L::coff(c), &maps.m[NF + c], &full_bar[s],
                        z0 - (halo_z(M, c) ? L::OFF : 0), y0 - (halo_y(M, c) ? R : 0), x);
#pragma unroll
          for (int q = 0; q < NP; ++q)
            tma_load_3d(st + NF * L::FRONT + L::CENTERS + q * L::FRONT,
                        &maps.m[NF + NC + q], &full_bar[s], z0, y0, x);
        }
      }
    }
    return;
  }

  const int z = z0 + V * lane;
  bool m0[RB], m1[RB];
#pragma unroll
  for (int j = 0; j < RB; ++j) {
    const bool yin = y0 + warp * RB + j < g.hi[1];
    m0[j] = yin && z >= g.lo[2] && z < g.hi[2];
    m1[j] = V > 1 && yin && z + 1 >= g.lo[2] && z + 1 < g.hi[2];
  }
  constexpr int W = 2 * R + 1;
  // x-windows unrolled by U planes: slots are constants inside the unrolled
  // group and the 2R live planes move down once per group (2R / U register
  // moves per plane instead of 2R; unroll_for)
  constexpr int U = unroll_for<Op, R>();
  T w[RB][NF > 0 ? NF : 1][W + U - 1];
#pragma unroll
  for (int j = 0; j < RB; ++j)
#pragma unroll
    for (int f = 0; f < NF; ++f)
#pragma unroll
      for (int k = 0; k < W + U - 1; ++k) w[j][f][k] = vconst<T>(0.f);

  for (int i0 = 0; i0 < nit; i0 += U) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u;
      if (i < nit) {
        const int s = i % L::S;
        mbar_wait(&full_bar[s], (i / L::S) & 1);
        const unsigned char* st = sm + s * L::STAGE;
#pragma unroll
        for (int j = 0; j < RB; ++j)
#pragma unroll
          for (int f = 0; f < NF; ++f)
            w[j][f][2 * R + u] = vload<V>(reinterpret_cast<const float*>(st + f * L::FRONT) +
                                          (warp * RB + j) * L::TZ + V * lane);
        if (i >= 2 * R) {
          const int x = xa + i - 2 * R;
#pragma unroll
          for (int j = 0; j < RB; ++j) {
            const int row = warp * RB + j, y = y0 + row;
            if (m0[j] || m1[j]) {
              StreamCtx<R, TY, V, NF, NC, NP, U, M> ctx{w[j], st, row, lane, u, &push, x, y, z};
              op.template point<R>(ctx, (int64_t)x * g.sx + (int64_t)y * g.sy + z, m0[j], m1[j]);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[s]);
      }
    }
#pragma unroll
    for (int j = 0; j < RB; ++j)
#pragma unroll
      for (int f = 0; f < NF; ++f)
#pragma unroll
        for (int k = 0; k < 2 * R; ++k) w[j][f][k] = w[j][f][k + U];
  }
}

// x-chunk count: whole waves of one CTA per SM, small priming overhead.
inline int stream_chunks(int64_t tiles, int nx, int R, int ctas = 1) {
  const int64_t slots = (int64_t)num_sms() * ctas;
  double best = 1e30;
  int best_n = 1;
  for (int n = 1; n <= 64 && n <= nx; ++n) {
    const int chunk = (nx + n - 1) / n;
    const int64_t items = tiles * ((nx + chunk - 1) / chunk);
    const int64_t waves = (items + slots - 1) / slots;
    const double cost = (double)waves * (chunk + 0.5 * 2 * R);
    if (cost < best - 1e-9) {
      best = cost;
      best_n = n;
    }
  }
  return best_n;
}

// Host launcher: `ptrs` = NF front arrays, then NC centre arrays, then NP
// point arrays (all FULL-shaped, same `full`).
template <int R, int TY, int V, class Op>
int launch_stream_op(const Op& op, const Geom& g, const int64_t full[3], const float* const* ptrs,
                     cudaStream_t st, const Push* push = nullptr) {
  using L = SLayout<R, TY, V, Op::NF, Op::NC, Op::NP, ctas_for<Op, TY>(), CHaloOf<Op>::value,
                    RowsOf<Op>::value, stages_for<Op, R>()>;
  static_assert(Op::NF + Op::NC + Op::NP <= kMaxMaps, "too many tensor maps");
  static int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    SDMP_CUDA(cudaFuncSetAttribute(stream_kernel<R, TY, V, Op>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, L::BYTES));
    attr_dev = dev;
  }
  TMaps maps;
  int k = 0;
  for (int f = 0; f < Op::NF; ++f, ++k) {
    int rc = make_tmap_3d(&maps.m[k], ptrs[k], full, L::TZ, TY, false);
    if (rc) return rc;
  }
  for (int c = 0; c < Op::NC; ++c, ++k) {
    int rc = make_tmap_3d(&maps.m[k], ptrs[k], full, L::cz(c), L::cy(c), false);
    if (rc) return rc;
  }
  for (int q = 0; q < Op::NP; ++q, ++k) {
    int rc = make_tmap_3d(&maps.m[k], ptrs[k], full, L::TZ, TY, true);
    if (rc) return rc;
  }
  const int nz = g.hi[2] - g.lo[2], ny = g.hi[1] - g.lo[1], nx = g.hi[0] - g.lo[0];
  const int tz = (nz + (g.lo[2] & 3) + L::TZ - 1) / L::TZ, ty = (ny + TY - 1) / TY;
  int nch = stream_chunks((int64_t)tz * ty, nx, R, ctas_for<Op, TY>());
  const int chunk = (nx + nch - 1) / nch;
  nch = (nx + chunk - 1) / chunk;
  SDMP_CHECK(nch <= 65535 && ty <= 65535, "grid too large");
  dim3 grid(tz, ty, nch), block(32, TY / RowsOf<Op>::value + 1);
  const bool dbg = getenv("SDMP_DEBUG") != nullptr;
  if (dbg)
    fprintf(stderr,
            "[sdmp] stream_kernel R=%d TY=%d V=%d NF=%d NC=%d NP=%d box=[%d,%d,%d]-[%d,%d,%d] "
            "full=[%ld,%ld,%ld] grid=(%d,%d,%d) chunk=%d smem=%d S=%d stage=%d\n",
            R, TY, V, Op::NF, Op::NC, Op::NP, g.lo[0], g.lo[1], g.lo[2], g.hi[0], g.hi[1],
            g.hi[2], (long)full[0], (long)full[1], (long)full[2], tz, ty, nch, chunk, L::BYTES,
            L::S, L::STAGE);
  const Push nopush{};
  stream_kernel<R, TY, V, Op><<<grid, block, L::BYTES, st>>>(maps, op, g, chunk,
                                                             push ? *push : nopush);
  SDMP_LAUNCHED();
  if (dbg) {
    cudaError_t e = cudaStreamSynchronize(st);
    fprintf(stderr, "[sdmp]   -> %s\n", cudaGetErrorString(e));
  }
  return SDMP_OK;
}

// TMA tile loads must start on a 16 B boundary along the innermost (z)
// axis: on sm_100a / driver 580 a misaligned box start raises "illegal
// instruction" (the engine aligns tiles down to 4 floats).  Loads start at
// (z0 - round4(R), y0 - R, x0 - R); boxes whose loads would start below 0
// take the generic kernel.
inline bool stream_fits(const Geom& g, int R) {
  return (g.lo[2] & ~3) - sround4(R) >= 0 && g.lo[1] - R >= 0 && g.lo[0] - R >= 0;
}

// TMA-eligibility of a set of arrays: 16 B-aligned bases, FULL z multiple of 4.
inline bool tma_ok(const int64_t full[3], const float* const* ptrs, int n) {
  if (full[2] % 4 != 0) return false;
  for (int i = 0; i < n; ++i)
    if (!ptrs[i] || (reinterpret_cast<uintptr_t>(ptrs[i]) & 15)) return false;
  return true;
}

}  // namespace sdmp
