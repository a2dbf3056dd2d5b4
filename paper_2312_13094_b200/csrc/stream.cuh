// Generic TMA streaming engine for multi-field stencils on sm_100a.
//
// A CTA owns a 32(z) x TY(y) tile and streams along x.  One producer warp
// fills an S-stage shared-memory ring with cp.async.bulk.tensor 3D tile
// loads (mbarrier complete_tx); TY consumer warps compute one point per
// thread (z = lane, y = warp).  Per pipeline iteration i (plane xa-R+i):
//
//   NF "front" tiles  [TY][32]              -> per-field x-window registers
//   NC "centre" tiles [TY+2R][32+2*OFF]     -> y / z taps (TMA zero-fills OOB)
//   NP "point" tiles  [TY][32]              -> pointwise operands
//
// front tiles run 2R planes ahead of the centre/point tiles, so at
// iteration i >= 2R the consumer holds planes x-R..x+R of every front field
// in registers and the centre/point tiles of plane x in the stage.
//
// The operator `Op` supplies
//   static constexpr int NF, NC, NP;
//   __device__ void point(const StreamCtx<...>&, int64_t idx) const;
// and the per-point arithmetic is shared with the one-thread-per-point
// generic kernels through accessor templates (bit-identical results).
#pragma once

#include <cstdio>
#include <cstdlib>

#include "tma.cuh"

namespace sdmp {

constexpr int kSZ = 32;  // z points per tile (one per lane)

__host__ __device__ constexpr int sround4(int r) { return (r + 3) & ~3; }

template <int R, int TY, int NF, int NC, int NP>
struct SLayout {
  static constexpr int OFF = sround4(R);
  static constexpr int CZ = kSZ + 2 * OFF;
  static constexpr int CY = TY + 2 * R;
  static constexpr int FRONT = kSZ * TY * 4;
  static constexpr int CENTER = ((CZ * CY * 4) + 127) & ~127;
  static constexpr int STAGE = NF * FRONT + NC * CENTER + NP * FRONT;
  static constexpr int S0 = (200 * 1024) / STAGE;
  static constexpr int S = S0 > 4 ? 4 : (S0 < 2 ? 2 : S0);
  static constexpr int BYTES = S * STAGE + 2 * S * 8 + 128;
  static constexpr int THREADS = 32 * (TY + 1);
  static constexpr uint32_t TX_FRONT = NF * FRONT;
  static constexpr uint32_t TX_MAIN = NF * FRONT + NC * CZ * CY * 4 + NP * FRONT;
};

constexpr int kMaxMaps = 24;
struct TMaps {
  CUtensorMap m[kMaxMaps];
};

// Consumer-side view of one point.
template <int R, int TY, int NF, int NC, int NP>
struct StreamCtx {
  using L = SLayout<R, TY, NF, NC, NP>;
  const float (*w)[2 * R + 1];   // x-windows
  const unsigned char* stage;
  int warp, lane;
  // field f (front index) at x + k
  __device__ __forceinline__ float xt(int f, int k) const { return w[f][R + k]; }
  // centre tile c at (y + dy, z + dz)
  __device__ __forceinline__ float ct(int c, int dy, int dz) const {
    const float* base = reinterpret_cast<const float*>(stage + NF * L::FRONT + c * L::CENTER);
    return base[(warp + R + dy) * L::CZ + L::OFF + lane + dz];
  }
  // point tile q
  __device__ __forceinline__ float pt(int q) const {
    const float* base = reinterpret_cast<const float*>(stage + NF * L::FRONT + NC * L::CENTER +
                                                       q * L::FRONT);
    return base[warp * kSZ + lane];
  }
};

template <int R, int TY, class Op>
__global__ void __launch_bounds__(SLayout<R, TY, Op::NF, Op::NC, Op::NP>::THREADS, 1)
stream_kernel(const __grid_constant__ TMaps maps, const Op op, const Geom g, const int xchunk) {
  constexpr int NF = Op::NF, NC = Op::NC, NP = Op::NP;
  using L = SLayout<R, TY, NF, NC, NP>;
  // __align__(1024) keeps TMA destinations aligned without integer pointer
  // arithmetic, so the compiler still sees shared-space pointers (LDS, not
  // generic LD) in the consumers
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = smraw;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(sm + L::S * L::STAGE);
  uint64_t* empty_bar = full_bar + L::S;
  const int lane = threadIdx.x, warp = threadIdx.y;
  if (lane == 0 && warp == 0) {
    for (int s = 0; s < L::S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], TY);
    }
    fence_barrier_init();
  }
  __syncthreads();
  // TMA boxes must start on a 16 B boundary along z: tiles are aligned down
  // to a multiple of 4 floats and lanes left of the box are masked off.
  const int z0 = (g.lo[2] & ~3) + blockIdx.x * kSZ;
  const int y0 = g.lo[1] + blockIdx.y * TY;
  const int xa = g.lo[0] + blockIdx.z * xchunk;
  const int xb = min(xa + xchunk, g.hi[0]);
  const int nit = (xb - xa) + 2 * R;

  if (warp == TY) {  // producer
    if (lane == 0) {
      for (int i = 0; i < nit; ++i) {
        const int s = i % L::S;
        mbar_wait(&empty_bar[s], ((i / L::S) & 1) ^ 1);
        unsigned char* st = sm + s * L::STAGE;
        const bool main = i >= 2 * R;
        mbar_arrive_expect_tx(&full_bar[s], main ? L::TX_MAIN : L::TX_FRONT);
        const int xf = xa - R + i;
#pragma unroll
        for (int f = 0; f < NF; ++f)
          tma_load_3d(st + f * L::FRONT, &maps.m[f], &full_bar[s], z0, y0, xf);
        if (main) {
          const int x = xa + i - 2 * R;
#pragma unroll
          for (int c = 0; c < NC; ++c)
            tma_load_3d(st + NF * L::FRONT + c * L::CENTER, &maps.m[NF + c], &full_bar[s],
                        z0 - L::OFF, y0 - R, x);
#pragma unroll
          for (int q = 0; q < NP; ++q)
            tma_load_3d(st + NF * L::FRONT + NC * L::CENTER + q * L::FRONT,
                        &maps.m[NF + NC + q], &full_bar[s], z0, y0, x);
        }
      }
    }
    return;
  }

  const int z = z0 + lane, y = y0 + warp;
  const bool active = (z >= g.lo[2]) && (z < g.hi[2]) && (y < g.hi[1]);
  float w[NF > 0 ? NF : 1][2 * R + 1];
#pragma unroll
  for (int f = 0; f < NF; ++f)
#pragma unroll
    for (int k = 0; k <= 2 * R; ++k) w[f][k] = 0.f;

  for (int i = 0; i < nit; ++i) {
    const int s = i % L::S;
    mbar_wait(&full_bar[s], (i / L::S) & 1);
    const unsigned char* st = sm + s * L::STAGE;
#pragma unroll
    for (int f = 0; f < NF; ++f) {
#pragma unroll
      for (int k = 0; k < 2 * R; ++k) w[f][k] = w[f][k + 1];
      w[f][2 * R] = reinterpret_cast<const float*>(st + f * L::FRONT)[warp * kSZ + lane];
    }
    if (i >= 2 * R && active) {
      const int x = xa + i - 2 * R;
      StreamCtx<R, TY, NF, NC, NP> ctx{w, st, warp, lane};
      op.template point<R>(ctx, (int64_t)x * g.sx + (int64_t)y * g.sy + z);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[s]);
  }
}

// x-chunk count: whole waves of one CTA per SM, small priming overhead.
inline int stream_chunks(int64_t tiles, int nx, int R) {
  const int64_t slots = (int64_t)num_sms();
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
template <int R, int TY, class Op>
int launch_stream_op(const Op& op, const Geom& g, const int64_t full[3], const float* const* ptrs,
                     cudaStream_t st) {
  using L = SLayout<R, TY, Op::NF, Op::NC, Op::NP>;
  static_assert(Op::NF + Op::NC + Op::NP <= kMaxMaps, "too many tensor maps");
  static int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    SDMP_CUDA(cudaFuncSetAttribute(stream_kernel<R, TY, Op>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, L::BYTES));
    attr_dev = dev;
  }
  TMaps maps;
  int k = 0;
  for (int f = 0; f < Op::NF; ++f, ++k) {
    int rc = make_tmap_3d(&maps.m[k], ptrs[k], full, kSZ, TY, false);
    if (rc) return rc;
  }
  for (int c = 0; c < Op::NC; ++c, ++k) {
    int rc = make_tmap_3d(&maps.m[k], ptrs[k], full, L::CZ, L::CY, false);
    if (rc) return rc;
  }
  for (int q = 0; q < Op::NP; ++q, ++k) {
    int rc = make_tmap_3d(&maps.m[k], ptrs[k], full, kSZ, TY, true);
    if (rc) return rc;
  }
  const int nz = g.hi[2] - g.lo[2], ny = g.hi[1] - g.lo[1], nx = g.hi[0] - g.lo[0];
  const int tz = (nz + (g.lo[2] & 3) + kSZ - 1) / kSZ, ty = (ny + TY - 1) / TY;
  int nch = stream_chunks((int64_t)tz * ty, nx, R);
  const int chunk = (nx + nch - 1) / nch;
  nch = (nx + chunk - 1) / chunk;
  SDMP_CHECK(nch <= 65535 && ty <= 65535, "grid too large");
  dim3 grid(tz, ty, nch), block(32, TY + 1);
  const bool dbg = getenv("SDMP_DEBUG") != nullptr;
  if (dbg)
    fprintf(stderr,
            "[sdmp] stream_kernel R=%d TY=%d NF=%d NC=%d NP=%d box=[%d,%d,%d]-[%d,%d,%d] "
            "full=[%ld,%ld,%ld] grid=(%d,%d,%d) chunk=%d smem=%d S=%d stage=%d\n",
            R, TY, Op::NF, Op::NC, Op::NP, g.lo[0], g.lo[1], g.lo[2], g.hi[0], g.hi[1], g.hi[2],
            (long)full[0], (long)full[1], (long)full[2], tz, ty, nch, chunk, L::BYTES, L::S,
            L::STAGE);
  stream_kernel<R, TY, Op><<<grid, block, L::BYTES, st>>>(maps, op, g, chunk);
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
