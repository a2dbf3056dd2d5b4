// Shared helpers for libsdmp (sm_100a).  See include/sdmp.h for the ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/sdmp.h"

namespace sdmp {

// Thread-local last error (sdmp_last_error).
void set_error(const std::string& msg);
const char* get_error();

#define SDMP_CUDA(call)                                                        \
  do {                                                                         \
    cudaError_t _e = (call);                                                   \
    if (_e != cudaSuccess) {                                                   \
      ::sdmp::set_error(std::string(#call) + ": " + cudaGetErrorString(_e) +   \
                        " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")"); \
      return SDMP_ECUDA;                                                       \
    }                                                                          \
  } while (0)

#define SDMP_CHECK(cond, msg)                                                  \
  do {                                                                         \
    if (!(cond)) {                                                             \
      ::sdmp::set_error(std::string("invalid argument: ") + (msg));            \
      return SDMP_EINVAL;                                                      \
    }                                                                          \
  } while (0)

#define SDMP_LAUNCHED()                                                        \
  do {                                                                         \
    cudaError_t _e = cudaGetLastError();                                       \
    if (_e != cudaSuccess) {                                                   \
      ::sdmp::set_error(std::string("kernel launch: ") + cudaGetErrorString(_e) + \
                        " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")"); \
      return SDMP_ECUDA;                                                       \
    }                                                                          \
  } while (0)

// Strided 3D geometry of one FULL array plus the box being computed.
struct Geom {
  int64_t sx, sy;        // element strides of x and y (z stride 1)
  int lo[3], hi[3];      // box, FULL coordinates, half-open
};

inline int make_geom(const int64_t full[3], const int64_t lo[3], const int64_t hi[3],
                     Geom* g) {
  for (int a = 0; a < 3; ++a) {
    SDMP_CHECK(full[a] > 0, "full shape must be positive");
    SDMP_CHECK(lo[a] >= 0 && hi[a] <= full[a], "box outside the FULL array");
    SDMP_CHECK(full[a] < (1ll << 31), "axis too long");
    g->lo[a] = (int)lo[a];
    g->hi[a] = (int)hi[a];
  }
  g->sy = full[2];
  g->sx = full[1] * full[2];
  return SDMP_OK;
}

// ---- fused halo push (full mode) -------------------------------------------
// A kernel that computes OWNED points also stores each result straight into
// the HALO of every neighbour whose receive box contains it (IPC-mapped peer
// pointers over NVLink): compute and halo exchange in ONE kernel.  For
// direction d, points of [lo, hi) (this rank's FULL coordinates) land at
// (x, y, z) + off in the peer's FULL array with strides (psx, psy, 1).
constexpr int kPushDirs = 8;
constexpr int kPushOut = 12;
struct PushGeo {
  int lo[3], hi[3], off[3];
  int64_t psx, psy;
};
struct Push {
  int ndir = 0, nout = 0;
  int64_t msx = 0, msy = 0;  // this rank's strides (inject decodes node indices)
  PushGeo geo[kPushDirs];
  float* base[kPushOut][kPushDirs];
};

__device__ __forceinline__ bool push_in(const PushGeo& g, int x, int y, int z) {
  return x >= g.lo[0] && x < g.hi[0] && y >= g.lo[1] && y < g.hi[1] && z >= g.lo[2] &&
         z < g.hi[2];
}

// one point, `nv` outputs (vals[q] -> base[q])
__device__ __forceinline__ void push_point(const Push& P, int x, int y, int z, const float* vals,
                                           int nv) {
  for (int d = 0; d < P.ndir; ++d) {
    const PushGeo& g = P.geo[d];
    if (!push_in(g, x, y, z)) continue;
    const int64_t j = (int64_t)(x + g.off[0]) * g.psx + (int64_t)(y + g.off[1]) * g.psy +
                      (z + g.off[2]);
    for (int q = 0; q < nv && q < P.nout; ++q)
      if (P.base[q][d]) P.base[q][d][j] = vals[q];
  }
}

// one box copy of a batched halo post (k_multi_copy)
struct CopyMsg {
  const float* src;
  float* dst;
  int64_t ssx, ssy, dsx, dsy, soff, doff;
  int ex, ey, ez;
};
constexpr int kMaxCopyMsgs = 96;
struct MultiCopy {
  int n = 0;
  int64_t rows = 0;
  int64_t row0[kMaxCopyMsgs];
  CopyMsg m[kMaxCopyMsgs];
};
int multi_copy(cudaStream_t st, const MultiCopy& mc);

inline bool box_empty(const Geom& g) {
  return g.hi[0] <= g.lo[0] || g.hi[1] <= g.lo[1] || g.hi[2] <= g.lo[2];
}

// CTA-partial barrier (bar.sync id, nthreads) for warp-specialised kernels
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

inline int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace sdmp
