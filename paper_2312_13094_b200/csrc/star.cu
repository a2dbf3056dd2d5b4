// Star-stencil family (acoustic SO 4..16, diffusion) for sm_100a.
//
// Replaces SPEC.md:311 compute(box, equation) for acoustic_kernel
// and diffusion_kernel.  The update is
// the reference's solved equation (symbolics.py:629-674) in the algebraic
// form u1 = A*u0 + B*u2 + S*L(u0), S = C/m or C, with the FD weights of
// fd_coefficients (symbolics.py:468-487) bound to fp32 once.
//
// Two kernels share ONE per-point evaluation sequence (star_point) written
// with explicit round-to-nearest intrinsics, so a point gets bit-identical
// results whichever kernel computes it: multi-rank runs (CORE by the
// streaming kernel, OWNED slabs by the generic one) equal single-rank runs
// bit for bit.
//
//  * star_generic: one thread per point, taps through L1/L2.  Any radius,
//    any alignment, 2D (radius_z = 0) included.  Used for thin OWNED slabs.
//  * star_tma<R,TY> / star_tma2<R,TY> / star_tmem<R,TY>: HBM-roofline kernels.  A CTA owns a
//    128(z) x TY(y) tile and streams along x (slowest axis); a producer warp
//    stages plane tiles with TMA, each consumer thread keeps a float4
//    x-window of 2R+1 planes in registers and reads y/z taps from the staged
//    centre plane (star_tmem: the x-window lives in tensor memory instead).
//    u0 is read from DRAM once (halo re-reads of neighbouring
//    tiles hit L2), u2 and m streamed once, u1 written once: 16 B / point.
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "stream.cuh"
#include "tma.cuh"
#include "tmem.cuh"
#include "vmath.cuh"

namespace sdmp {

#ifndef SDMP_STAR_TMEM_MINR
#define SDMP_STAR_TMEM_MINR 7  // smallest radius on the TMEM x-window kernel (r04 A/B)
#endif
// Front tiles are loaded with an L2 evict_last hint: R planes later the same
// rows come back as the centre tile's interior and as the neighbouring
// tiles' y halo.  r04 A/B (1024^3): star_tmem SO-16 +2.2% (DRAM 1.147x ->
// 1.108x algorithmic), SO-14 +1.9%, star_tma2 SO-12 +0.5%, SO-4/8 neutral;
// hinting the centre / pointwise tiles evict_first as well lost
// (profiles/round2_ab_front_l2.txt).
#ifndef SDMP_TMA_L2
#define SDMP_TMA_L2 1
#endif

struct StarParams {
  const float* __restrict__ u0;
  const float* __restrict__ u2;
  const float* __restrict__ m;
  float* __restrict__ u1;
  Geom g;
  int r[3];
  float c[3][SDMP_NCOEF];
  float csum0;  // c_x0 + c_y0 + c_z0 (fp32, host-rounded)
  float A, B, C;
  int m_is_scale;  // m holds the bound scale S = C/m (sdmp_bind_scale)
  // variable-coefficient family (sdmp_var_star_update): per-point A and B
  // (B may be null); S comes through m with m_is_scale = 1
  const float* __restrict__ Av;
  const float* __restrict__ Bv;
};

// Shared tail of the per-point update: u1 = A*u0 + B*u2 + S*lap.
__device__ __forceinline__ float star_finish(const StarParams& p, float lap, float c0, float u2v,
                                             float mv, float av, float bv) {
  float s = (p.m == nullptr) ? p.C : (p.m_is_scale ? mv : __fdiv_rn(p.C, mv));
  float t = __fmul_rn(av, c0);
  t = __fmaf_rn(bv, u2v, t);
  return __fmaf_rn(s, lap, t);
}
__device__ __forceinline__ float star_finish(const StarParams& p, float lap, float c0, float u2v,
                                             float mv) {
  return star_finish(p, lap, c0, u2v, mv, p.A, p.B);
}

// Per-point update.  xs(k)/ys(k)/zs(k) return tap(-k) + tap(+k) along the
// axis; the sum is formed with __fadd_rn inside the caller.
template <int RX, int RY, int RZ, class FX, class FY, class FZ>
__device__ __forceinline__ float star_point(const StarParams& p, float c0, float u2v, float mv,
                                            int rx, int ry, int rz, FX xs, FY ys, FZ zs,
                                            float av, float bv) {
  float lap = __fmul_rn(p.csum0, c0);
#pragma unroll
  for (int k = 1; k <= (RX > 0 ? RX : SDMP_MAX_RADIUS); ++k)
    if (RX > 0 || k <= rx) lap = __fmaf_rn(p.c[0][k], xs(k), lap);
#pragma unroll
  for (int k = 1; k <= (RY > 0 ? RY : SDMP_MAX_RADIUS); ++k)
    if (RY > 0 || k <= ry) lap = __fmaf_rn(p.c[1][k], ys(k), lap);
#pragma unroll
  for (int k = 1; k <= (RZ > 0 ? RZ : SDMP_MAX_RADIUS); ++k)
    if (RZ > 0 || k <= rz) lap = __fmaf_rn(p.c[2][k], zs(k), lap);
  return star_finish(p, lap, c0, u2v, mv, av, bv);
}

// ---------------------------------------------------------------------------
// generic: one thread per point

__global__ void __launch_bounds__(256) star_generic(StarParams p, const Push push) {
  const int z = p.g.lo[2] + blockIdx.x * 32 + threadIdx.x;
  const int y = p.g.lo[1] + blockIdx.y * 8 + threadIdx.y;
  const int x = p.g.lo[0] + blockIdx.z;
  if (z >= p.g.hi[2] || y >= p.g.hi[1]) return;
  const int64_t sx = p.g.sx, sy = p.g.sy;
  const int64_t i = x * sx + y * sy + z;
  const float* __restrict__ u = p.u0;
  float c0 = __ldg(u + i);
  float u2v = p.u2 ? __ldg(p.u2 + i) : 0.0f;
  float mv = p.m ? __ldg(p.m + i) : 1.0f;
  auto xs = [&](int k) { return __fadd_rn(__ldg(u + i - k * sx), __ldg(u + i + k * sx)); };
  auto ys = [&](int k) { return __fadd_rn(__ldg(u + i - k * sy), __ldg(u + i + k * sy)); };
  auto zs = [&](int k) { return __fadd_rn(__ldg(u + i - k), __ldg(u + i + k)); };
  const float av = p.Av ? __ldg(p.Av + i) : p.A;
  const float bv = p.Av ? (p.Bv ? __ldg(p.Bv + i) : 0.0f) : p.B;
  const float v = star_point<0, 0, 0>(p, c0, u2v, mv, p.r[0], p.r[1], p.r[2], xs, ys, zs, av, bv);
  p.u1[i] = v;
  if (push.ndir) push_point(push, x, y, z, &v, 1);
}

// ---------------------------------------------------------------------------
// streaming kernels: tile width along z

constexpr int kTZ = 128;  // z points per tile (32 lanes x float4)

__host__ __device__ constexpr int round4(int r) { return (r + 3) & ~3; }

// lanes (x, y) or (z, w) of a float4 as one packed pair
__device__ __forceinline__ V2 f4pair(const float4& v, int h) {
  return h == 0 ? v2pack(v.x, v.y) : v2pack(v.z, v.w);
}
__device__ __forceinline__ float f4get(const float4& v, int j) {
  return j == 0 ? v.x : j == 1 ? v.y : j == 2 ? v.z : v.w;
}

// ---------------------------------------------------------------------------
// TMA pipeline: one producer warp streams plane tiles into an S-stage shared
// ring with cp.async.bulk.tensor (mbarrier complete_tx); TY consumer warps
// (one y row each, float4 along z) keep the x-window in registers and read
// y/z taps from the staged centre plane.  No __syncthreads in the loop.
//
// Per pipeline iteration i (plane p = xa - R + i):
//   front  [TY][128]            u0 at plane p         -> register window
//   centre [TY+2R][128+2*OFF]   u0 at plane p-R (=x)  -> y/z taps   (i >= 2R)
//   u2, m  [TY][128]            at plane x                          (i >= 2R)

// ---- pieces shared by the TMA star kernels (one row of 4 z points) -------

// z taps of one row: zw = the row's z neighbourhood (OFF floats each side)
template <int R, int OFF>
__device__ __forceinline__ void star_ztaps(const StarParams& p, const float* zw, V2 lap[2]) {
#pragma unroll
  for (int k = 1; k <= R; ++k) {
    if ((k & 1) == 0) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int lo = OFF + 2 * h - k, hi = OFF + 2 * h + k;
        lap[h] = vcfma(p.c[2][k], vadd(v2pack(zw[lo], zw[lo + 1]), v2pack(zw[hi], zw[hi + 1])),
                       lap[h]);
      }
    } else {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int lo = OFF + 2 * h - k, hi = OFF + 2 * h + k;
        const float l0 = __fmaf_rn(p.c[2][k], __fadd_rn(zw[lo], zw[hi]), v2lo(lap[h]));
        const float l1 = __fmaf_rn(p.c[2][k], __fadd_rn(zw[lo + 1], zw[hi + 1]), v2hi(lap[h]));
        lap[h] = v2pack(l0, l1);
      }
    }
  }
}

// z neighbourhood of a thread's 4 points (zw[0 .. 4 + 2 OFF), centred at OFF):
// SDMP_ZSHFL = 1 takes the thread's own 4 values from its x-window register
// (the centre plane) and the neighbours' from the adjacent lanes' registers
// by warp shuffles; only lanes at the warp's edge read the staged halo
// columns.  0 reads the whole neighbourhood from the staged centre row
// (NZW 16-byte loads).  Same values either way.  All 32 lanes must call it.
#ifndef SDMP_ZSHFL
#define SDMP_ZSHFL 0
#endif
template <int OFF>
__device__ __forceinline__ void star_zwin(float* zw, const float4& own, const float* row,
                                          int lane) {
  constexpr int NZW = (4 + 2 * OFF) / 4;
#if SDMP_ZSHFL
  zw[OFF + 0] = own.x; zw[OFF + 1] = own.y; zw[OFF + 2] = own.z; zw[OFF + 3] = own.w;
#pragma unroll
  for (int t = 1; t <= OFF / 4; ++t) {
    float4 lo, hi;
    lo.x = __shfl_up_sync(0xffffffffu, own.x, t);
    lo.y = __shfl_up_sync(0xffffffffu, own.y, t);
    lo.z = __shfl_up_sync(0xffffffffu, own.z, t);
    lo.w = __shfl_up_sync(0xffffffffu, own.w, t);
    hi.x = __shfl_down_sync(0xffffffffu, own.x, t);
    hi.y = __shfl_down_sync(0xffffffffu, own.y, t);
    hi.z = __shfl_down_sync(0xffffffffu, own.z, t);
    hi.w = __shfl_down_sync(0xffffffffu, own.w, t);
    if (lane < t) lo = *reinterpret_cast<const float4*>(row - 4 * t);
    if (lane + t > 31) hi = *reinterpret_cast<const float4*>(row + 4 * t);
    const int l0 = OFF - 4 * t, h0 = OFF + 4 * t;
    zw[l0 + 0] = lo.x; zw[l0 + 1] = lo.y; zw[l0 + 2] = lo.z; zw[l0 + 3] = lo.w;
    zw[h0 + 0] = hi.x; zw[h0 + 1] = hi.y; zw[h0 + 2] = hi.z; zw[h0 + 3] = hi.w;
  }
  (void)NZW;
#else
  (void)own;
  (void)lane;
#pragma unroll
  for (int q = 0; q < NZW; ++q) {
    const float4 v = *reinterpret_cast<const float4*>(row - OFF + 4 * q);
    zw[4 * q + 0] = v.x; zw[4 * q + 1] = v.y; zw[4 * q + 2] = v.z; zw[4 * q + 3] = v.w;
  }
#endif
}

// u1 = A u0 + B u2 + S lap on 4 points (star_finish per lane)
__device__ __forceinline__ void star_finish4(const StarParams& p, const V2 lap[2], const float4& c0,
                                             const float4& u2v, const float4& mv, float out[4]) {
  if (p.m == nullptr || p.m_is_scale) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const V2 sc = p.m == nullptr ? v2bcast(p.C) : f4pair(mv, h);
      V2 t = vcmul(p.A, f4pair(c0, h));
      t = vcfma(p.B, f4pair(u2v, h), t);
      const V2 o = vfma(sc, lap[h], t);
      out[2 * h] = v2lo(o);
      out[2 * h + 1] = v2hi(o);
    }
  } else {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      out[2 * h] = star_finish(p, v2lo(lap[h]), f4get(c0, 2 * h), f4get(u2v, 2 * h),
                               f4get(mv, 2 * h));
      out[2 * h + 1] = star_finish(p, v2hi(lap[h]), f4get(c0, 2 * h + 1), f4get(u2v, 2 * h + 1),
                                   f4get(mv, 2 * h + 1));
    }
  }
}

// streaming store of 4 points + fused halo push: the float4 also lands in
// every neighbour HALO whose receive box contains it
__device__ __forceinline__ void star_store4(const StarParams& p, const Push& push, int x, int y,
                                            int z, const float out[4]) {
  __stcs(reinterpret_cast<float4*>(p.u1 + (int64_t)x * p.g.sx + (int64_t)y * p.g.sy + z),
         make_float4(out[0], out[1], out[2], out[3]));
  for (int d = 0; d < push.ndir; ++d) {
    const PushGeo& pg = push.geo[d];
    if (x < pg.lo[0] || x >= pg.hi[0] || y < pg.lo[1] || y >= pg.hi[1] || z + 3 < pg.lo[2] ||
        z >= pg.hi[2])
      continue;
    float* dst = push.base[0][d] + (int64_t)(x + pg.off[0]) * pg.psx +
                 (int64_t)(y + pg.off[1]) * pg.psy + (z + pg.off[2]);
    if (z >= pg.lo[2] && z + 3 < pg.hi[2] && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
      *reinterpret_cast<float4*>(dst) = make_float4(out[0], out[1], out[2], out[3]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (z + j >= pg.lo[2] && z + j < pg.hi[2]) dst[j] = out[j];
    }
  }
}

template <int R, int TY>
struct TmaCfg {
  static constexpr int OFF = round4(R);
  static constexpr int CZ = kTZ + 2 * OFF;
  static constexpr int CY = TY + 2 * R;
  static constexpr int FRONT = kTZ * TY * 4;
  static constexpr int CENTER = ((CZ * CY * 4) + 127) & ~127;
  static constexpr int STAGE = 3 * FRONT + CENTER;
#ifndef SDMP_STAR_STAGES
#define SDMP_STAR_STAGES 4
#endif
  // pipeline depth: SDMP_STAR_STAGES planes in flight, fewer if they do not fit
  static constexpr int S0 = (224 * 1024 - 2048) / STAGE;
  static constexpr int S = SDMP_STAR_STAGES < S0 ? SDMP_STAR_STAGES : S0;
  static constexpr int BYTES = S * STAGE + 2 * S * 8 + 128;
  static constexpr int THREADS = 32 * (TY + 1);
};

// x-window as an unrolled register ring (no per-plane register moves) for
// the wide stencils; SDMP_STAR_RING_MIN sets the smallest radius using it
// the x-window of star_tma is an unrolled register ring up to R = 4 (r02
// A/B: wider stencils lose to code size); star_tma2 unrolls its x-windows
// by two planes (r03 A/B) and runs 14-row tiles at R = 8 (8 warps, 208
// registers; 12 and 16 rows measured slower).  (r04 A/B, dropped: one
// accumulation chain per axis instead of one per point -- SO-16 unchanged,
// SO-12 -2%, the damped SO-16 stream op -25%.)
constexpr int kTma2Unroll = 2;
constexpr int kTma2RowsR8 = 14;

template <int R>
constexpr bool kStarRing = R >= 1 && R <= 4;

template <int R, int TY>
__global__ void __launch_bounds__(TmaCfg<R, TY>::THREADS, 1)
star_tma(const __grid_constant__ CUtensorMap tm_front, const __grid_constant__ CUtensorMap tm_center,
         const __grid_constant__ CUtensorMap tm_u2, const __grid_constant__ CUtensorMap tm_m,
         StarParams p, int xchunk, const Push push) {
  using T = TmaCfg<R, TY>;
  // __align__(1024) keeps TMA destinations aligned without integer pointer
  // arithmetic, so the compiler still sees shared-space pointers (LDS, not
  // generic LD) in the consumers
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = smraw;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(sm + T::S * T::STAGE);
  uint64_t* empty_bar = full_bar + T::S;
  const int lane = threadIdx.x, warp = threadIdx.y;
  const bool has_u2 = p.u2 != nullptr, has_m = p.m != nullptr;
  if (lane == 0 && warp == 0) {
    for (int s = 0; s < T::S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], TY);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int z0 = p.g.lo[2] + blockIdx.x * kTZ;
  const int y0 = p.g.lo[1] + blockIdx.y * TY;
  const int xa = p.g.lo[0] + blockIdx.z * xchunk;
  const int xb = min(xa + xchunk, p.g.hi[0]);
  const int nit = (xb - xa) + 2 * R;

  if (warp == TY) {  // producer
    if (lane == 0) {
      prefetch_tmap(&tm_front);
      prefetch_tmap(&tm_center);
      const uint32_t main_bytes =
          T::FRONT + T::CZ * T::CY * 4 + (has_u2 ? T::FRONT : 0) + (has_m ? T::FRONT : 0);
      for (int i = 0; i < nit; ++i) {
        const int s = i % T::S;
        mbar_wait(&empty_bar[s], ((i / T::S) & 1) ^ 1);
        unsigned char* st = sm + s * T::STAGE;
        const bool main = i >= 2 * R;
        mbar_arrive_expect_tx(&full_bar[s], main ? main_bytes : (uint32_t)T::FRONT);
#if SDMP_TMA_L2
        tma_load_3d_hint(st, &tm_front, &full_bar[s], z0, y0, xa - R + i, l2_policy_evict_last());
#else
        tma_load_3d(st, &tm_front, &full_bar[s], z0, y0, xa - R + i);
#endif
        if (main) {
          const int x = xa + i - 2 * R;
          tma_load_3d(st + T::FRONT, &tm_center, &full_bar[s], z0 - T::OFF, y0 - R, x);
          if (has_u2) tma_load_3d(st + T::FRONT + T::CENTER, &tm_u2, &full_bar[s], z0, y0, x);
          if (has_m)
            tma_load_3d(st + 2 * T::FRONT + T::CENTER, &tm_m, &full_bar[s], z0, y0, x);
        }
      }
    }
    return;
  }

  const int z = z0 + 4 * lane, y = y0 + warp;
  const bool active = (z < p.g.hi[2]) && (y < p.g.hi[1]);
  constexpr int W = 2 * R + 1;
  float4 w[W];
#pragma unroll
  for (int k = 0; k < W; ++k) w[k] = make_float4(0.f, 0.f, 0.f, 0.f);

  // one pipeline iteration; the x-window plane of logical index kk (0 =
  // oldest, 2R = newest) sits in register slot (rot + kk + 1) % W
  const bool yact = y < p.g.hi[1];  // warp-uniform (one row per warp)
  auto consume = [&](int i, int rot, const unsigned char* st) {
    auto wv = [&](int kk) -> const float4& { return w[(rot + kk + 1) % W]; };
    if (i >= 2 * R && yact) {  // every lane of the warp (shuffles), stores masked
      const int x = xa + i - 2 * R;
      const float* row = reinterpret_cast<const float*>(st + T::FRONT) + (warp + R) * T::CZ +
                         T::OFF + 4 * lane;
      constexpr int NZW = (4 + 2 * T::OFF) / 4;
      float zw[4 * NZW];
      star_zwin<T::OFF>(zw, wv(R), row, lane);
      float4 u2v = make_float4(0.f, 0.f, 0.f, 0.f), mv = make_float4(1.f, 1.f, 1.f, 1.f);
      if (has_u2)
        u2v = *reinterpret_cast<const float4*>(
            reinterpret_cast<const float*>(st + T::FRONT + T::CENTER) + warp * kTZ + 4 * lane);
      if (has_m)
        mv = *reinterpret_cast<const float4*>(
            reinterpret_cast<const float*>(st + 2 * T::FRONT + T::CENTER) + warp * kTZ + 4 * lane);
      // same operation order per point as star_point (x, y, z taps; k
      // ascending), on the 4 z points of this thread as two packed fp32x2
      // pairs (FFMA2 / FADD2: per-lane IEEE ops, identical bits).  Odd z
      // shifts straddle the register pairs, so those taps run per lane.
      V2 lap[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) lap[h] = vcmul(p.csum0, f4pair(wv(R), h));
#pragma unroll
      for (int k = 1; k <= R; ++k)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          lap[h] = vcfma(p.c[0][k], vadd(f4pair(wv(R - k), h), f4pair(wv(R + k), h)), lap[h]);
#pragma unroll
      for (int k = 1; k <= R; ++k) {
        const float4 a = *reinterpret_cast<const float4*>(row - k * T::CZ);
        const float4 b = *reinterpret_cast<const float4*>(row + k * T::CZ);
#pragma unroll
        for (int h = 0; h < 2; ++h)
          lap[h] = vcfma(p.c[1][k], vadd(f4pair(a, h), f4pair(b, h)), lap[h]);
      }
      star_ztaps<R, T::OFF>(p, zw, lap);
      float out[4];
      star_finish4(p, lap, wv(R), u2v, mv, out);
      if (active) star_store4(p, push, x, y, z, out);
    }
  };

  if constexpr (kStarRing<R>) {
    // register ring: unrolled by W, slot indices are constants (no moves)
    for (int i0 = 0; i0 < nit; i0 += W) {
#pragma unroll
      for (int j = 0; j < W; ++j) {
        const int i = i0 + j;
        if (i < nit) {
          const int s = i % T::S;
          mbar_wait(&full_bar[s], (i / T::S) & 1);
          const unsigned char* st = sm + s * T::STAGE;
          w[j] = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(st) +
                                                  warp * kTZ + 4 * lane);
          consume(i, j, st);
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty_bar[s]);
        }
      }
    }
  } else {
    for (int i = 0; i < nit; ++i) {
      const int s = i % T::S;
      mbar_wait(&full_bar[s], (i / T::S) & 1);
      const unsigned char* st = sm + s * T::STAGE;
#pragma unroll
      for (int k = 0; k < 2 * R; ++k) w[k] = w[k + 1];
      w[2 * R] = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(st) +
                                                  warp * kTZ + 4 * lane);
      consume(i, W - 1, st);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[s]);
    }
  }
}

// Pick the number of x chunks: whole waves of one CTA per SM, small
// priming overhead (2R front-only iterations per chunk).
// cost of n x-chunks = waves x (chunk planes + x-window fill + per-CTA fixed
// cost `cta_planes`, in plane units).  star_tma: 4 planes (prologue, tensor-map
// prefetch, pipeline fill / drain) -- at C1's 256^3 one wave of 64-plane-chunk
// CTAs beats two waves of 29-plane chunks by 5% (profiles/r03_ab_nch.log);
// 512^3 and 1024^3 keep their choices.
static int pick_chunks(int64_t tiles, int nx, int R, int ctas_per_sm, double cta_planes = 0.0) {
  const int64_t slots = (int64_t)num_sms() * ctas_per_sm;
  double best = 1e30;
  int best_n = 1;
  for (int n = 1; n <= 64 && n <= nx; ++n) {
    const int chunk = (nx + n - 1) / n;
    const int64_t items = tiles * ((nx + chunk - 1) / chunk);
    const int64_t waves = (items + slots - 1) / slots;
    const double cost = (double)waves * (chunk + 0.35 * 2 * R + cta_planes);
    if (cost < best - 1e-9) {
      best = cost;
      best_n = n;
    }
  }
  return best_n;
}

template <int R, int TY>
static int launch_tma(const StarParams& p, cudaStream_t st, const int64_t full[3],
                      const Push& push, int ctas = 1) {
  using T = TmaCfg<R, TY>;
  static int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    SDMP_CUDA(cudaFuncSetAttribute(star_tma<R, TY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   T::BYTES));
    attr_dev = dev;
  }
  CUtensorMap tf, tc, t2, tm;
  int rc = make_tmap_3d(&tf, p.u0, full, kTZ, TY, false);
  if (!rc) rc = make_tmap_3d(&tc, p.u0, full, T::CZ, T::CY, false);
  if (!rc) rc = make_tmap_3d(&t2, p.u2 ? p.u2 : p.u0, full, kTZ, TY, true);
  if (!rc) rc = make_tmap_3d(&tm, p.m ? p.m : p.u0, full, kTZ, TY, true);
  if (rc) return rc;
  const int nz = p.g.hi[2] - p.g.lo[2], ny = p.g.hi[1] - p.g.lo[1], nx = p.g.hi[0] - p.g.lo[0];
  const int tz = (nz + kTZ - 1) / kTZ, ty = (ny + TY - 1) / TY;
  int nch = pick_chunks((int64_t)tz * ty, nx, R, ctas, 4.0);
  const int chunk = (nx + nch - 1) / nch;
  nch = (nx + chunk - 1) / chunk;
  SDMP_CHECK(nch <= 65535 && ty <= 65535, "grid too large");
  dim3 grid(tz, ty, nch), block(32, TY + 1);
  star_tma<R, TY><<<grid, block, T::BYTES, st>>>(tf, tc, t2, tm, p, chunk, push);
  SDMP_LAUNCHED();
  return SDMP_OK;
}

// ---------------------------------------------------------------------------
// Wide stencils (R >= 6): the same pipeline with TWO consecutive y rows per
// consumer thread.  The 2R+2 staged rows a thread needs for both rows' y taps
// are read from shared memory once (software-pipelined so each row keeps its
// k-ascending order): 34 instead of 48 LDS.128 per 8 points, and TY = 16 rows
// per CTA halves the centre tile's y-halo overhead versus one row per warp
// (the wide stencils are shared-memory-bandwidth bound, profiles/r02).

template <int R, int TY>
__global__ void __launch_bounds__(32 * (TY / 2 + 1), 1)
star_tma2(const __grid_constant__ CUtensorMap tm_front, const __grid_constant__ CUtensorMap tm_center,
          const __grid_constant__ CUtensorMap tm_u2, const __grid_constant__ CUtensorMap tm_m,
          StarParams p, int xchunk, const Push push) {
  using T = TmaCfg<R, TY>;
  constexpr int NW = TY / 2;  // consumer warps
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = smraw;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(sm + T::S * T::STAGE);
  uint64_t* empty_bar = full_bar + T::S;
  const int lane = threadIdx.x, warp = threadIdx.y;
  const bool has_u2 = p.u2 != nullptr, has_m = p.m != nullptr;
  if (lane == 0 && warp == 0) {
    for (int s = 0; s < T::S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], NW);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int z0 = p.g.lo[2] + blockIdx.x * kTZ;
  const int y0 = p.g.lo[1] + blockIdx.y * TY;
  const int xa = p.g.lo[0] + blockIdx.z * xchunk;
  const int xb = min(xa + xchunk, p.g.hi[0]);
  const int nit = (xb - xa) + 2 * R;

  if (warp == NW) {  // producer
    if (lane == 0) {
      prefetch_tmap(&tm_front);
      prefetch_tmap(&tm_center);
      const uint32_t main_bytes =
          T::FRONT + T::CZ * T::CY * 4 + (has_u2 ? T::FRONT : 0) + (has_m ? T::FRONT : 0);
      for (int i = 0; i < nit; ++i) {
        const int s = i % T::S;
        mbar_wait(&empty_bar[s], ((i / T::S) & 1) ^ 1);
        unsigned char* st = sm + s * T::STAGE;
        const bool main = i >= 2 * R;
        mbar_arrive_expect_tx(&full_bar[s], main ? main_bytes : (uint32_t)T::FRONT);
#if SDMP_TMA_L2
        tma_load_3d_hint(st, &tm_front, &full_bar[s], z0, y0, xa - R + i, l2_policy_evict_last());
#else
        tma_load_3d(st, &tm_front, &full_bar[s], z0, y0, xa - R + i);
#endif
        if (main) {
          const int x = xa + i - 2 * R;
          tma_load_3d(st + T::FRONT, &tm_center, &full_bar[s], z0 - T::OFF, y0 - R, x);
          if (has_u2) tma_load_3d(st + T::FRONT + T::CENTER, &tm_u2, &full_bar[s], z0, y0, x);
          if (has_m)
            tma_load_3d(st + 2 * T::FRONT + T::CENTER, &tm_m, &full_bar[s], z0, y0, x);
        }
      }
    }
    return;
  }

  const int z = z0 + 4 * lane, r0 = 2 * warp;  // rows r0, r0 + 1 of the tile
  const bool zin = z < p.g.hi[2];
  const bool act0 = zin && (y0 + r0 < p.g.hi[1]), act1 = zin && (y0 + r0 + 1 < p.g.hi[1]);
  constexpr int W = 2 * R + 1;
  // x-windows unrolled by U planes: plane slots are constants inside the
  // unrolled group and the 2R live planes move down once per group (2R / U
  // register moves per plane instead of 2R; r03 A/B)
  constexpr int U = kTma2Unroll;
  float4 w0[W + U - 1], w1[W + U - 1];
#pragma unroll
  for (int k = 0; k < W + U - 1; ++k) w0[k] = w1[k] = make_float4(0.f, 0.f, 0.f, 0.f);

  // one x-plane: window slots b .. b + 2R (b = group position, a constant)
  const bool ract = y0 + r0 < p.g.hi[1];  // warp-uniform: the warp's first row
  auto consume = [&](const int i, const int b, const unsigned char* st) {
    if (i >= 2 * R && ract) {  // every lane of the warp (shuffles), stores masked
      const int x = xa + i - 2 * R;
      // centre tile row (r0 + R + d) at this thread's 4 z points
      const float* crow = reinterpret_cast<const float*>(st + T::FRONT) + (r0 + R) * T::CZ +
                          T::OFF + 4 * lane;
      auto rowv = [&](int d) { return *reinterpret_cast<const float4*>(crow + d * T::CZ); };
      V2 l0[2], l1[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        l0[h] = vcmul(p.csum0, f4pair(w0[b + R], h));
        l1[h] = vcmul(p.csum0, f4pair(w1[b + R], h));
      }
#pragma unroll
      for (int k = 1; k <= R; ++k)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          l0[h] = vcfma(p.c[0][k], vadd(f4pair(w0[b + R - k], h), f4pair(w0[b + R + k], h)), l0[h]);
          l1[h] = vcfma(p.c[0][k], vadd(f4pair(w1[b + R - k], h), f4pair(w1[b + R + k], h)), l1[h]);
        }
      // y taps: row 0 uses rows -k / +k, row 1 rows 1-k / 1+k (k ascending
      // for each): A_k = row(-k), B_k = row(+k); row 1 at k takes
      // A_{k-1} (A_0 = row 0) and B_{k+1}, loaded one step ahead
      float4 am = rowv(0), bk = rowv(1), bn;
#pragma unroll
      for (int k = 1; k <= R; ++k) {
        const float4 ak = rowv(-k);
        bn = rowv(k + 1);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          l0[h] = vcfma(p.c[1][k], vadd(f4pair(ak, h), f4pair(bk, h)), l0[h]);
          l1[h] = vcfma(p.c[1][k], vadd(f4pair(am, h), f4pair(bn, h)), l1[h]);
        }
        am = ak;
        bk = bn;
      }
      constexpr int NZW = (4 + 2 * T::OFF) / 4;
      float zw[4 * NZW];
      float out[4];
      const float* pts = reinterpret_cast<const float*>(st + T::FRONT + T::CENTER) + 4 * lane;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        star_zwin<T::OFF>(zw, j == 0 ? w0[b + R] : w1[b + R], crow + j * T::CZ, lane);
        V2* l = j == 0 ? l0 : l1;
        star_ztaps<R, T::OFF>(p, zw, l);
        const int rr = r0 + j;
        const float4 u2v = has_u2 ? *reinterpret_cast<const float4*>(pts + rr * kTZ)
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 mv = has_m ? *reinterpret_cast<const float4*>(pts + T::FRONT / 4 + rr * kTZ)
                                : make_float4(1.f, 1.f, 1.f, 1.f);
        star_finish4(p, l, j == 0 ? w0[b + R] : w1[b + R], u2v, mv, out);
        if (j == 0 ? act0 : act1) star_store4(p, push, x, y0 + rr, z, out);
      }
    }
  };

  for (int i0 = 0; i0 < nit; i0 += U) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u;
      if (i < nit) {
        const int s = i % T::S;
        mbar_wait(&full_bar[s], (i / T::S) & 1);
        const unsigned char* st = sm + s * T::STAGE;
        const float* front = reinterpret_cast<const float*>(st) + 4 * lane;
        w0[2 * R + u] = *reinterpret_cast<const float4*>(front + r0 * kTZ);
        w1[2 * R + u] = *reinterpret_cast<const float4*>(front + (r0 + 1) * kTZ);
        consume(i, u, st);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[s]);
      }
    }
#pragma unroll
    for (int k = 0; k < 2 * R; ++k) {
      w0[k] = w0[k + U];
      w1[k] = w1[k + U];
    }
  }
}

template <int R, int TY>
static int launch_tma2(const StarParams& p, cudaStream_t st, const int64_t full[3],
                       const Push& push) {
  using T = TmaCfg<R, TY>;
  static int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    SDMP_CUDA(cudaFuncSetAttribute(star_tma2<R, TY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   T::BYTES));
    attr_dev = dev;
  }
  CUtensorMap tf, tc, t2, tm;
  int rc = make_tmap_3d(&tf, p.u0, full, kTZ, TY, false);
  if (!rc) rc = make_tmap_3d(&tc, p.u0, full, T::CZ, T::CY, false);
  if (!rc) rc = make_tmap_3d(&t2, p.u2 ? p.u2 : p.u0, full, kTZ, TY, true);
  if (!rc) rc = make_tmap_3d(&tm, p.m ? p.m : p.u0, full, kTZ, TY, true);
  if (rc) return rc;
  const int nz = p.g.hi[2] - p.g.lo[2], ny = p.g.hi[1] - p.g.lo[1], nx = p.g.hi[0] - p.g.lo[0];
  const int tz = (nz + kTZ - 1) / kTZ, ty = (ny + TY - 1) / TY;
  int nch = pick_chunks((int64_t)tz * ty, nx, R, 1);
  const int chunk = (nx + nch - 1) / nch;
  nch = (nx + chunk - 1) / chunk;
  SDMP_CHECK(nch <= 65535 && ty <= 65535, "grid too large");
  dim3 grid(tz, ty, nch), block(32, TY / 2 + 1);
  star_tma2<R, TY><<<grid, block, T::BYTES, st>>>(tf, tc, t2, tm, p, chunk, push);
  SDMP_LAUNCHED();
  return SDMP_OK;
}

// ---------------------------------------------------------------------------
// Widest stencils: star_tma2's pipeline with the x-window in TENSOR MEMORY.
// At R = 8 the two 17-plane register windows (144 registers) pin star_tma2
// to 8 warps per SM, where it is latency bound (profiles/r03_unroll.md).
// Here the window is a ring of 2R plane slots in TMEM: each consumer thread
// owns 8 columns per slot (its 2 rows x 4 z points) of its warp's lane
// quarter.  Per plane a thread reads the 2R - 1 older planes back with
// tcgen05.ld (64 B / point, ~a quarter of TMEM read bandwidth at the HBM
// roofline), takes the centre plane from the staged centre tile and the
// newest plane from the front tile, and writes the newest plane into the
// slot the oldest one just vacated.  Registers drop to ~100, so TY / 2 = 12
// consumer warps run per SM.  Arithmetic is star_tma2's, term for term.
#ifndef SDMP_TMEM_KC
#define SDMP_TMEM_KC 4  // x-tap pairs per tcgen05.ld batch
#endif
#ifndef SDMP_TMEM_ROWS
#define SDMP_TMEM_ROWS 24
#endif
template <int R, int TY>
struct TmemCfg {
  static constexpr int NW = TY / 2;                 // consumer warps
  static constexpr int SLICES = (NW + 3) / 4;       // warps sharing a lane quarter
  static constexpr int SLOT = 8;                    // columns per plane slot
  static constexpr int COLS_USED = SLICES * 2 * R * SLOT;
  static constexpr int COLS = COLS_USED <= 128 ? 128 : COLS_USED <= 256 ? 256 : 512;
  static_assert(COLS_USED <= 512, "x-window ring does not fit TMEM");
};

template <int R, int TY>
__global__ void __launch_bounds__(32 * (TY / 2 + 1), 1)
star_tmem(const __grid_constant__ CUtensorMap tm_front, const __grid_constant__ CUtensorMap tm_center,
          const __grid_constant__ CUtensorMap tm_u2, const __grid_constant__ CUtensorMap tm_m,
          StarParams p, int xchunk, const Push push) {
  using T = TmaCfg<R, TY>;
  using M = TmemCfg<R, TY>;
  constexpr int NW = M::NW;
  constexpr int KC = SDMP_TMEM_KC;
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = smraw;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(sm + T::S * T::STAGE);
  uint64_t* empty_bar = full_bar + T::S;
  uint32_t* tbase = reinterpret_cast<uint32_t*>(empty_bar + T::S);
  const int lane = threadIdx.x, warp = threadIdx.y;
  const bool has_u2 = p.u2 != nullptr, has_m = p.m != nullptr;
  if (lane == 0 && warp == 0) {
    for (int s = 0; s < T::S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], NW);
    }
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<M::COLS>(tbase);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const int z0 = p.g.lo[2] + blockIdx.x * kTZ;
  const int y0 = p.g.lo[1] + blockIdx.y * TY;
  const int xa = p.g.lo[0] + blockIdx.z * xchunk;
  const int xb = min(xa + xchunk, p.g.hi[0]);
  const int nit = (xb - xa) + 2 * R;

  if (warp == NW) {  // producer
    if (lane == 0) {
      prefetch_tmap(&tm_front);
      prefetch_tmap(&tm_center);
      const uint32_t main_bytes =
          T::FRONT + T::CZ * T::CY * 4 + (has_u2 ? T::FRONT : 0) + (has_m ? T::FRONT : 0);
      for (int i = 0; i < nit; ++i) {
        const int s = i % T::S;
        mbar_wait(&empty_bar[s], ((i / T::S) & 1) ^ 1);
        unsigned char* st = sm + s * T::STAGE;
        const bool main = i >= 2 * R;
        mbar_arrive_expect_tx(&full_bar[s], main ? main_bytes : (uint32_t)T::FRONT);
#if SDMP_TMA_L2
        tma_load_3d_hint(st, &tm_front, &full_bar[s], z0, y0, xa - R + i, l2_policy_evict_last());
#else
        tma_load_3d(st, &tm_front, &full_bar[s], z0, y0, xa - R + i);
#endif
        if (main) {
          const int x = xa + i - 2 * R;
          tma_load_3d(st + T::FRONT, &tm_center, &full_bar[s], z0 - T::OFF, y0 - R, x);
          if (has_u2) tma_load_3d(st + T::FRONT + T::CENTER, &tm_u2, &full_bar[s], z0, y0, x);
          if (has_m)
            tma_load_3d(st + 2 * T::FRONT + T::CENTER, &tm_m, &full_bar[s], z0, y0, x);
        }
      }
    }
    return;
  }

  const int z = z0 + 4 * lane, r0 = 2 * warp;  // rows r0, r0 + 1 of the tile
  const bool zin = z < p.g.hi[2];
  const bool act0 = zin && (y0 + r0 < p.g.hi[1]), act1 = zin && (y0 + r0 + 1 < p.g.hi[1]);
  const bool ract = y0 + r0 < p.g.hi[1];  // warp-uniform
  // this warp's ring: lane quarter warp % 4, column slice warp / 4
  const uint32_t ring = *tbase + (static_cast<uint32_t>(32 * (warp & 3)) << 16) +
                        static_cast<uint32_t>((warp >> 2) * 2 * R * M::SLOT);
  auto slot_addr = [&](int s) { return ring + static_cast<uint32_t>(s * M::SLOT); };

  for (int i = 0; i < nit; ++i) {
    const int s = i % T::S;
    mbar_wait(&full_bar[s], (i / T::S) & 1);
    const unsigned char* st = sm + s * T::STAGE;
    if (ract) {
      tmem_wait_st();  // last plane's slot write has landed (and freed its registers)
      const float* front = reinterpret_cast<const float*>(st) + 4 * lane;
      const float4 fa = *reinterpret_cast<const float4*>(front + r0 * kTZ);
      const float4 fb = *reinterpret_cast<const float4*>(front + (r0 + 1) * kTZ);
      const int snew = i % (2 * R);  // slot of this iteration's newest plane
      if (i >= 2 * R) {
        const int x = xa + i - 2 * R;
        const float* crow = reinterpret_cast<const float*>(st + T::FRONT) + (r0 + R) * T::CZ +
                            T::OFF + 4 * lane;
        auto rowv = [&](int d) { return *reinterpret_cast<const float4*>(crow + d * T::CZ); };
        const float4 c0a = rowv(0), c0b = rowv(1);
        V2 l0[2], l1[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          l0[h] = vcmul(p.csum0, f4pair(c0a, h));
          l1[h] = vcmul(p.csum0, f4pair(c0b, h));
        }
        // x taps: planes x -/+ k live in slots (scen -/+ k) mod 2R, scen =
        // the centre plane's slot; x + R (slot scen + R = snew) is the front
        const int scen = (i - R) % (2 * R);
#pragma unroll
        for (int k0 = 1; k0 <= R; k0 += KC) {
          float4 ma[KC], mb[KC], pa[KC], pb[KC];
#pragma unroll
          for (int j = 0; j < KC; ++j) {
            const int k = k0 + j;
            if (k > R) break;
            int sm_ = scen - k;
            sm_ += sm_ < 0 ? 2 * R : 0;
            tmem_ld8(slot_addr(sm_), ma[j], mb[j]);
            if (k < R) {
              int sp = scen + k;
              sp -= sp >= 2 * R ? 2 * R : 0;
              tmem_ld8(slot_addr(sp), pa[j], pb[j]);
            }
          }
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < KC; ++j) {
            const int k = k0 + j;
            if (k > R) break;
            tmem_pin(ma[j]);
            tmem_pin(mb[j]);
            if (k < R) {
              tmem_pin(pa[j]);
              tmem_pin(pb[j]);
            } else {
              pa[j] = fa;
              pb[j] = fb;
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              l0[h] = vcfma(p.c[0][k], vadd(f4pair(ma[j], h), f4pair(pa[j], h)), l0[h]);
              l1[h] = vcfma(p.c[0][k], vadd(f4pair(mb[j], h), f4pair(pb[j], h)), l1[h]);
            }
          }
        }
        // the oldest plane (x - R) has been read: its slot takes the newest
        tmem_st8(slot_addr(snew), fa, fb);
        // y taps (star_tma2's software-pipelined pairs)
        float4 am = c0a, bk = c0b, bn;
#pragma unroll
        for (int k = 1; k <= R; ++k) {
          const float4 ak = rowv(-k);
          bn = rowv(k + 1);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            l0[h] = vcfma(p.c[1][k], vadd(f4pair(ak, h), f4pair(bk, h)), l0[h]);
            l1[h] = vcfma(p.c[1][k], vadd(f4pair(am, h), f4pair(bn, h)), l1[h]);
          }
          am = ak;
          bk = bn;
        }
        constexpr int NZW = (4 + 2 * T::OFF) / 4;
        float zw[4 * NZW];
        float out[4];
        const float* pts = reinterpret_cast<const float*>(st + T::FRONT + T::CENTER) + 4 * lane;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          star_zwin<T::OFF>(zw, j == 0 ? c0a : c0b, crow + j * T::CZ, lane);
          V2* l = j == 0 ? l0 : l1;
          star_ztaps<R, T::OFF>(p, zw, l);
          const int rr = r0 + j;
          const float4 u2v = has_u2 ? *reinterpret_cast<const float4*>(pts + rr * kTZ)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
          const float4 mv = has_m ? *reinterpret_cast<const float4*>(pts + T::FRONT / 4 + rr * kTZ)
                                  : make_float4(1.f, 1.f, 1.f, 1.f);
          star_finish4(p, l, j == 0 ? c0a : c0b, u2v, mv, out);
          if (j == 0 ? act0 : act1) star_store4(p, push, x, y0 + rr, z, out);
        }
      } else {
        tmem_st8(slot_addr(snew), fa, fb);  // filling the ring
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[s]);
  }
  tmem_wait_st();
  tmem_fence_before();
  named_sync(1, NW * 32);
  tmem_fence_after();
  if (warp == 0) tmem_dealloc<M::COLS>(*tbase);
}

template <int R, int TY>
static int launch_tmem(const StarParams& p, cudaStream_t st, const int64_t full[3],
                       const Push& push) {
  using T = TmaCfg<R, TY>;
  constexpr int BYTES = T::BYTES + 16;  // + the TMEM base address
  static int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    SDMP_CUDA(cudaFuncSetAttribute(star_tmem<R, TY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   BYTES));
    attr_dev = dev;
  }
  CUtensorMap tf, tc, t2, tm;
  int rc = make_tmap_3d(&tf, p.u0, full, kTZ, TY, false);
  if (!rc) rc = make_tmap_3d(&tc, p.u0, full, T::CZ, T::CY, false);
  if (!rc) rc = make_tmap_3d(&t2, p.u2 ? p.u2 : p.u0, full, kTZ, TY, true);
  if (!rc) rc = make_tmap_3d(&tm, p.m ? p.m : p.u0, full, kTZ, TY, true);
  if (rc) return rc;
  const int nz = p.g.hi[2] - p.g.lo[2], ny = p.g.hi[1] - p.g.lo[1], nx = p.g.hi[0] - p.g.lo[0];
  const int tz = (nz + kTZ - 1) / kTZ, ty = (ny + TY - 1) / TY;
  int nch = pick_chunks((int64_t)tz * ty, nx, R, 1);
  const int chunk = (nx + nch - 1) / nch;
  nch = (nx + chunk - 1) / chunk;
  SDMP_CHECK(nch <= 65535 && ty <= 65535, "grid too large");
  dim3 grid(tz, ty, nch), block(32, TY / 2 + 1);
  star_tmem<R, TY><<<grid, block, BYTES, st>>>(tf, tc, t2, tm, p, chunk, push);
  SDMP_LAUNCHED();
  return SDMP_OK;
}

// ---------------------------------------------------------------------------
// variable-coefficient star on the generic TMA stream engine: fronts {u0},
// centre {u0}, points {u2 (if B), A, B (if present), S}; same per-point order
// as star_point + star_finish
#ifndef SDMP_VSTAR_CTAS
#define SDMP_VSTAR_CTAS 1
#endif
template <bool HAS_B>
struct VarStarOp {
  static constexpr int NF = 1, NC = 1, NP = HAS_B ? 4 : 2;
  static constexpr int kCtas = SDMP_VSTAR_CTAS;
  StarParams p{};
  template <int R, class Ctx>
  __device__ __forceinline__ void point(const Ctx& c, int64_t idx, bool m0, bool m1) const {
    using T = typename Ctx::T;
    const T c0 = c.xt(0, 0);
    T lap = vcmul(p.csum0, c0);
#pragma unroll
    for (int k = 1; k <= R; ++k) lap = vcfma(p.c[0][k], vadd(c.xt(0, -k), c.xt(0, k)), lap);
#pragma unroll
    for (int k = 1; k <= R; ++k) lap = vcfma(p.c[1][k], vadd(c.ct(0, -k, 0), c.ct(0, k, 0)), lap);
#pragma unroll
    for (int k = 1; k <= R; ++k) lap = vcfma(p.c[2][k], vadd(c.ct(0, 0, -k), c.ct(0, 0, k)), lap);
    const T u2v = HAS_B ? c.pt(0) : vconst<T>(0.f);
    const T av = c.pt(HAS_B ? 1 : 0);
    const T bv = HAS_B ? c.pt(2) : vconst<T>(0.f);
    const T sv = c.pt(HAS_B ? 3 : 1);
    T t = vmul(av, c0);
    t = vfma(bv, u2v, t);
    const T o = vfma(sv, lap, t);
    vstore(p.u1, idx, o, m0, m1);
    c.push_out(&o, 1, m0, m1);
  }
};

template <int R>
static int launch_var_engine(const StarParams& p, cudaStream_t st, const int64_t full[3],
                             const Push& push) {
#ifndef SDMP_VSTAR_TYN
#define SDMP_VSTAR_TYN 16
#endif
#ifndef SDMP_VSTAR_TYW
#define SDMP_VSTAR_TYW 8
#endif
  constexpr int TY = R <= 4 ? SDMP_VSTAR_TYN : SDMP_VSTAR_TYW;
  if (p.Bv) {
    VarStarOp<true> op{};
    op.p = p;
    const float* arrs[6] = {p.u0, p.u0, p.u2, p.Av, p.Bv, p.m};
    return launch_stream_op<R, TY, 2>(op, p.g, full, arrs, st, &push);
  }
  VarStarOp<false> op{};
  op.p = p;
  const float* arrs[4] = {p.u0, p.u0, p.Av, p.m};
  return launch_stream_op<R, TY, 2>(op, p.g, full, arrs, st, &push);
}

static int launch_generic(const StarParams& p, cudaStream_t st, const Push& push) {
  const int nz = p.g.hi[2] - p.g.lo[2], ny = p.g.hi[1] - p.g.lo[1], nx = p.g.hi[0] - p.g.lo[0];
  SDMP_CHECK(nx <= 65535, "generic kernel: box x extent > 65535");
  dim3 block(32, 8);
  dim3 grid((nz + 31) / 32, (ny + 7) / 8, nx);
  star_generic<<<grid, block, 0, st>>>(p, push);
  SDMP_LAUNCHED();
  return SDMP_OK;
}

int star_update(cudaStream_t st, const float* u0, const float* u2, const float* m, float* u1,
                const int64_t full[3], const int64_t lo[3], const int64_t hi[3],
                const int32_t radius[3], const float* coeffs, float A, float B, float C,
                int variant, const Push* push_in) {
  const Push nopush{};
  const Push& push = push_in ? *push_in : nopush;
  StarParams p{};
  int rc = make_geom(full, lo, hi, &p.g);
  if (rc) return rc;
  SDMP_CHECK(u0 && u1, "u0/u1 must be non-null");
  SDMP_CHECK(B == 0.0f || u2, "u2 required when B != 0");
  if (box_empty(p.g)) return SDMP_OK;
  p.u0 = u0; p.u2 = (B == 0.0f) ? nullptr : u2; p.m = m; p.u1 = u1;
  p.m_is_scale = (variant & SDMP_VARIANT_M_IS_SCALE) ? 1 : 0;
  variant &= 0xff;
  if (variant == 0) {  // SDMP_STAR_VARIANT (tests): 1 generic, 3 one-row TMA at every R,
                       // 4 register-window two-row TMA at R >= 6
    const char* e = getenv("SDMP_STAR_VARIANT");
    variant = e ? atoi(e) : 0;
  }
  float cs = 0.f;
  for (int a = 0; a < 3; ++a) {
    SDMP_CHECK(radius[a] >= 0 && radius[a] <= SDMP_MAX_RADIUS, "radius outside 0..8");
    SDMP_CHECK(lo[a] >= radius[a] && hi[a] + radius[a] <= full[a], "box + radius exceeds FULL");
    p.r[a] = radius[a];
    for (int k = 0; k < SDMP_NCOEF; ++k) p.c[a][k] = (k <= radius[a]) ? coeffs[a * SDMP_NCOEF + k] : 0.f;
    cs = cs + p.c[a][0];  // (cx0 + cy0) + cz0
  }
  p.csum0 = cs;
  p.A = A; p.B = B; p.C = C;

  const int R = radius[0];
  const bool streamable = radius[1] == R && radius[2] == R && R >= 1 && lo[2] >= round4(R) &&
                          (full[2] % 4 == 0) && (lo[2] % 4 == 0) && ((hi[2] - lo[2]) % 4 == 0) &&
                          (((uintptr_t)u0 | (uintptr_t)u1 | (uintptr_t)u2 | (uintptr_t)m) % 16 == 0);
  if (getenv("SDMP_DEBUG"))
    fprintf(stderr, "[sdmp] star_update R=%d box=[%ld,%ld,%ld]-[%ld,%ld,%ld] %s push=%d\n", R,
            (long)lo[0], (long)lo[1], (long)lo[2], (long)hi[0], (long)hi[1], (long)hi[2],
            (variant == 1 || !streamable) ? "generic"
            : (variant == 0 && R >= SDMP_STAR_TMEM_MINR) ? "star_tmem"
            : ((variant == 0 || variant == 4) && R >= 6) ? "star_tma2" : "star_tma",
            push.ndir);
  // unaligned / unequal-radius boxes always take the generic kernel
  if (variant == 1 || !streamable) return launch_generic(p, st, push);
  // wide stencils: two rows per thread.  R >= 7: x-window in tensor memory
  // (star_tmem, 24-row tiles, 12 consumer warps at 104 registers): SO-16
  // 0.716 -> 0.846 and SO-14 0.794 -> 0.884 of the HBM roofline, SO-12 keeps
  // the register window (0.936 vs 0.917; profiles/round2_ab_tmem.txt).
  // star_tma2: 16-row tiles (9 warps: ptxas caps registers at 168) while the
  // two x-windows fit; R = 8 needs ~210 registers, so 14-row tiles (8 warps)
  if (variant == 0 && R >= SDMP_STAR_TMEM_MINR) {
    switch (R) {
      case 6: return launch_tmem<6, SDMP_TMEM_ROWS>(p, st, full, push);
      case 7: return launch_tmem<7, SDMP_TMEM_ROWS>(p, st, full, push);
      case 8: return launch_tmem<8, SDMP_TMEM_ROWS>(p, st, full, push);
    }
  }
  if (variant == 0 || variant == 4) {  // 4 (tests): register-window star_tma2
    switch (R) {
      case 6: return launch_tma2<6, 16>(p, st, full, push);
      case 7: return launch_tma2<7, 16>(p, st, full, push);
      case 8: return launch_tma2<8, kTma2RowsR8>(p, st, full, push);
    }
  }
  switch (R) {  // variant 0 (auto) / 3: TMA pipeline
    case 1: return launch_tma<1, 16>(p, st, full, push);
    case 2: return launch_tma<2, 16>(p, st, full, push);
    case 3: return launch_tma<3, 16>(p, st, full, push);
    case 4: return launch_tma<4, 16>(p, st, full, push);
    case 5: return launch_tma<5, 16>(p, st, full, push);
    case 6: return launch_tma<6, 8>(p, st, full, push);
    case 7: return launch_tma<7, 8>(p, st, full, push);
    case 8: return launch_tma<8, 8>(p, st, full, push);
  }
  return launch_generic(p, st, push);
}

int var_star_update(cudaStream_t st, const float* u0, const float* u2, const float* A,
                    const float* B, const float* Sarr, float* u1, const int64_t full[3],
                    const int64_t lo[3], const int64_t hi[3], const int32_t radius[3],
                    const float* coeffs, int variant, const Push* push_in) {
  const Push nopush{};
  const Push& push = push_in ? *push_in : nopush;
  StarParams p{};
  int rc = make_geom(full, lo, hi, &p.g);
  if (rc) return rc;
  SDMP_CHECK(u0 && u1 && A && Sarr, "u0, u1, A and S must be non-null");
  SDMP_CHECK(!B || u2, "u2 required with B");
  if (box_empty(p.g)) return SDMP_OK;
  p.u0 = u0; p.u2 = B ? u2 : nullptr; p.m = Sarr; p.u1 = u1; p.Av = A; p.Bv = B;
  p.m_is_scale = 1;
  p.A = 0.f; p.B = 0.f; p.C = 1.f;
  if ((variant & 0xff) == 0) {  // SDMP_STAR_VARIANT=1 (tests): the generic kernel
    const char* e = getenv("SDMP_STAR_VARIANT");
    if (e && atoi(e) == 1) variant = 1;
  }
  float cs = 0.f;
  for (int a = 0; a < 3; ++a) {
    SDMP_CHECK(radius[a] >= 0 && radius[a] <= SDMP_MAX_RADIUS, "radius outside 0..8");
    SDMP_CHECK(lo[a] >= radius[a] && hi[a] + radius[a] <= full[a], "box + radius exceeds FULL");
    p.r[a] = radius[a];
    for (int k = 0; k < SDMP_NCOEF; ++k) p.c[a][k] = (k <= radius[a]) ? coeffs[a * SDMP_NCOEF + k] : 0.f;
    cs = cs + p.c[a][0];
  }
  p.csum0 = cs;
  const int R = radius[0];
  if ((variant & 0xff) != 1 && radius[1] == R && radius[2] == R && R >= 1) {
    const float* arrs[6] = {u0, u1, u2 ? u2 : u0, A, B ? B : A, Sarr};
    Geom g = p.g;
    if (stream_fits(g, R) && tma_ok(full, arrs, 6)) {
      switch (R) {
        case 1: return launch_var_engine<1>(p, st, full, push);
        case 2: return launch_var_engine<2>(p, st, full, push);
        case 3: return launch_var_engine<3>(p, st, full, push);
        case 4: return launch_var_engine<4>(p, st, full, push);
        case 5: return launch_var_engine<5>(p, st, full, push);
        case 6: return launch_var_engine<6>(p, st, full, push);
        case 7: return launch_var_engine<7>(p, st, full, push);
        case 8: return launch_var_engine<8>(p, st, full, push);
      }
    }
  }
  return launch_generic(p, st, push);
}

}  // namespace sdmp

extern "C" int sdmp_var_star_update(void* stream, const float* u0, const float* u2,
                                    const float* A, const float* B, const float* S, float* u1,
                                    const int64_t full[3], const int64_t lo[3],
                                    const int64_t hi[3], const int32_t radius[3],
                                    const float* coeffs, int32_t variant) {
  return sdmp::var_star_update((cudaStream_t)stream, u0, u2, A, B, S, u1, full, lo, hi, radius,
                               coeffs, variant, nullptr);
}

extern "C" int sdmp_star_update(void* stream, const float* u0, const float* u2, const float* m,
                                float* u1, const int64_t full[3], const int64_t lo[3],
                                const int64_t hi[3], const int32_t radius[3],
                                const float* coeffs, float A, float B, float C,
                                int32_t variant) {
  return sdmp::star_update((cudaStream_t)stream, u0, u2, m, u1, full, lo, hi, radius, coeffs,
                           A, B, C, variant, nullptr);
}
