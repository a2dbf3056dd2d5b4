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
// Two passes per box: tti_g writes g(p), g(r) on the box grown by R into a
// FULL-shaped scratch pair; tti_update applies the outer derivative.  The
// per-point arithmetic is fixed (explicit _rn intrinsics) so CORE/OWNED/
// DOMAIN launches agree bit for bit.
#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"

namespace sdmp {

struct TTIParams {
  const float* __restrict__ p0;
  const float* __restrict__ p2;
  const float* __restrict__ r0;
  const float* __restrict__ r2;
  const float* __restrict__ m;
  const float* __restrict__ epsp;
  const float* __restrict__ delp;
  const float* __restrict__ a[3];
  float* __restrict__ gp;
  float* __restrict__ gr;
  float* __restrict__ p1;
  float* __restrict__ r1;
  Geom g;
  int R;
  float lap[3][SDMP_NCOEF];
  float d1[3][SDMP_NCOEF];
  float csum0;
  float dt2;
};

template <int R>
__device__ __forceinline__ float dcentral(const float* __restrict__ f, int64_t i, int64_t s,
                                          const float* w) {
  float acc = __fmul_rn(w[1], __fsub_rn(__ldg(f + i + s), __ldg(f + i - s)));
#pragma unroll
  for (int k = 2; k <= R; ++k)
    acc = __fmaf_rn(w[k], __fsub_rn(__ldg(f + i + k * s), __ldg(f + i - k * s)), acc);
  return acc;
}

template <int R>
__global__ void __launch_bounds__(256) tti_g(TTIParams p, int glo0, int glo1, int glo2,
                                             int ghi0, int ghi1, int ghi2) {
  const int z = glo2 + blockIdx.x * 32 + threadIdx.x;
  const int y = glo1 + blockIdx.y * 8 + threadIdx.y;
  const int x = glo0 + blockIdx.z;
  if (z >= ghi2 || y >= ghi1 || x >= ghi0) return;
  const int64_t s[3] = {p.g.sx, p.g.sy, 1};
  const int64_t i = x * s[0] + y * s[1] + z;
  float ax = __ldg(p.a[0] + i), ay = __ldg(p.a[1] + i), az = __ldg(p.a[2] + i);
  float gpv = __fmul_rn(ax, dcentral<R>(p.p0, i, s[0], p.d1[0]));
  gpv = __fmaf_rn(ay, dcentral<R>(p.p0, i, s[1], p.d1[1]), gpv);
  gpv = __fmaf_rn(az, dcentral<R>(p.p0, i, s[2], p.d1[2]), gpv);
  float grv = __fmul_rn(ax, dcentral<R>(p.r0, i, s[0], p.d1[0]));
  grv = __fmaf_rn(ay, dcentral<R>(p.r0, i, s[1], p.d1[1]), grv);
  grv = __fmaf_rn(az, dcentral<R>(p.r0, i, s[2], p.d1[2]), grv);
  p.gp[i] = gpv;
  p.gr[i] = grv;
}

template <int R>
__device__ __forceinline__ float outer(const float* __restrict__ a, const float* __restrict__ g,
                                       int64_t i, int64_t s, const float* w) {
  float acc = 0.f;
#pragma unroll
  for (int k = 1; k <= R; ++k) {
    float hi = __fmul_rn(__ldg(a + i + k * s), g[i + k * s]);
    float lo = __fmul_rn(__ldg(a + i - k * s), g[i - k * s]);
    acc = k == 1 ? __fmul_rn(w[1], __fsub_rn(hi, lo)) : __fmaf_rn(w[k], __fsub_rn(hi, lo), acc);
  }
  return acc;
}

template <int R>
__global__ void __launch_bounds__(256) tti_update(TTIParams p) {
  const int z = p.g.lo[2] + blockIdx.x * 32 + threadIdx.x;
  const int y = p.g.lo[1] + blockIdx.y * 8 + threadIdx.y;
  const int x = p.g.lo[0] + blockIdx.z;
  if (z >= p.g.hi[2] || y >= p.g.hi[1]) return;
  const int64_t s[3] = {p.g.sx, p.g.sy, 1};
  const int64_t i = x * s[0] + y * s[1] + z;
  float gzp = outer<R>(p.a[0], p.gp, i, s[0], p.d1[0]);
  gzp = __fadd_rn(gzp, outer<R>(p.a[1], p.gp, i, s[1], p.d1[1]));
  gzp = __fadd_rn(gzp, outer<R>(p.a[2], p.gp, i, s[2], p.d1[2]));
  float gzr = outer<R>(p.a[0], p.gr, i, s[0], p.d1[0]);
  gzr = __fadd_rn(gzr, outer<R>(p.a[1], p.gr, i, s[1], p.d1[1]));
  gzr = __fadd_rn(gzr, outer<R>(p.a[2], p.gr, i, s[2], p.d1[2]));
  const float* __restrict__ u = p.p0;
  float c0 = __ldg(u + i);
  float lap = __fmul_rn(p.csum0, c0);
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int k = 1; k <= R; ++k)
      lap = __fmaf_rn(p.lap[a][k], __fadd_rn(__ldg(u + i - k * s[a]), __ldg(u + i + k * s[a])), lap);
  float h0 = __fsub_rn(lap, gzp);
  float sc = __fdiv_rn(p.dt2, __ldg(p.m + i));
  float e = __ldg(p.epsp + i), d = __ldg(p.delp + i);
  float pp = __fmaf_rn(d, gzr, __fmul_rn(e, h0));
  float rr = __fmaf_rn(d, h0, gzr);
  float pt = __fsub_rn(__fmul_rn(2.f, c0), __ldg(p.p2 + i));
  float r0v = __ldg(p.r0 + i);
  float rt = __fsub_rn(__fmul_rn(2.f, r0v), __ldg(p.r2 + i));
  p.p1[i] = __fmaf_rn(sc, pp, pt);
  p.r1[i] = __fmaf_rn(sc, rr, rt);
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
  if (cudaMalloc(&b, n * sizeof(float)) != cudaSuccess) { cudaFree(a); return {nullptr, nullptr}; }
  cudaMemset(a, 0, n * sizeof(float));
  cudaMemset(b, 0, n * sizeof(float));
  cache[key] = {a, b};
  return {a, b};
}

// R = first-derivative radius (SO/2); the nested operator reaches 2R.
template <int R>
static int launch(TTIParams& p, cudaStream_t st) {
  int glo[3], ghi[3];
  for (int a = 0; a < 3; ++a) {
    glo[a] = p.g.lo[a] - R;
    ghi[a] = p.g.hi[a] + R;
  }
  dim3 b(32, 8);
  dim3 g1((ghi[2] - glo[2] + 31) / 32, (ghi[1] - glo[1] + 7) / 8, ghi[0] - glo[0]);
  tti_g<R><<<g1, b, 0, st>>>(p, glo[0], glo[1], glo[2], ghi[0], ghi[1], ghi[2]);
  SDMP_LAUNCHED();
  dim3 g2((p.g.hi[2] - p.g.lo[2] + 31) / 32, (p.g.hi[1] - p.g.lo[1] + 7) / 8,
          p.g.hi[0] - p.g.lo[0]);
  tti_update<R><<<g2, b, 0, st>>>(p);
  SDMP_LAUNCHED();
  return SDMP_OK;
}

int tti_update_entry(cudaStream_t st, const float* const in[10], float* p1, float* r1,
                     const int64_t full[3], const int64_t lo[3], const int64_t hi[3],
                     int32_t radius, const float* lap_c, const float* d1_c, float dt2) {
  TTIParams p;
  int rc = make_geom(full, lo, hi, &p.g);
  if (rc) return rc;
  if (box_empty(p.g)) return SDMP_OK;
  SDMP_CHECK(radius >= 1 && radius <= SDMP_MAX_RADIUS, "tti radius (SO/2) outside 1..8");
  for (int i = 0; i < 10; ++i) SDMP_CHECK(in[i] != nullptr, "tti inputs must be non-null");
  for (int a = 0; a < 3; ++a)
    SDMP_CHECK(lo[a] >= 2 * radius && hi[a] + 2 * radius <= full[a],
               "tti box + 2*radius exceeds FULL (halo must be >= SO)");
  p.p0 = in[0]; p.p2 = in[1]; p.r0 = in[2]; p.r2 = in[3]; p.m = in[4];
  p.epsp = in[5]; p.delp = in[6]; p.a[0] = in[7]; p.a[1] = in[8]; p.a[2] = in[9];
  p.p1 = p1; p.r1 = r1;
  p.R = radius;
  float cs = 0.f;
  for (int a = 0; a < 3; ++a) {
    for (int k = 0; k < SDMP_NCOEF; ++k) {
      p.lap[a][k] = k <= radius ? lap_c[a * SDMP_NCOEF + k] : 0.f;
      p.d1[a][k] = (k >= 1 && k <= radius) ? d1_c[a * SDMP_NCOEF + k] : 0.f;
    }
    cs = cs + p.lap[a][0];
  }
  p.csum0 = cs;
  p.dt2 = dt2;
  auto sc = scratch(full[0] * full[1] * full[2]);
  if (!sc.first) {
    set_error("tti: scratch allocation failed");
    return SDMP_ECUDA;
  }
  p.gp = sc.first;
  p.gr = sc.second;
  switch (radius) {
    case 1: return launch<1>(p, st);
    case 2: return launch<2>(p, st);
    case 3: return launch<3>(p, st);
    case 4: return launch<4>(p, st);
    case 5: return launch<5>(p, st);
    case 6: return launch<6>(p, st);
    case 7: return launch<7>(p, st);
    case 8: return launch<8>(p, st);
  }
  set_error("tti: unsupported radius");
  return SDMP_EUNSUPPORTED;
}

}  // namespace sdmp

extern "C" int sdmp_tti_update(void* stream, const float* const in[10], float* p1, float* r1,
                               const int64_t full[3], const int64_t lo[3], const int64_t hi[3],
                               int32_t radius, const float* lap_c, const float* d1_c, float dt2,
                               int32_t variant) {
  (void)variant;
  return sdmp::tti_update_entry((cudaStream_t)stream, in, p1, r1, full, lo, hi, radius, lap_c,
                                d1_c, dt2);
}
