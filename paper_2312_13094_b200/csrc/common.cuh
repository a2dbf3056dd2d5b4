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

inline bool box_empty(const Geom& g) {
  return g.hi[0] <= g.lo[0] || g.hi[1] <= g.lo[1] || g.hi[2] <= g.lo[2];
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
