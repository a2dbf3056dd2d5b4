// Staggered-grid velocity-stress elastic and single-relaxation
// viscoelastic kernels for sm_100a.
//
// Replaces compute(box, equation) of elastic_kernel (here
// on the paper's staggered grid, weights from staggered_coefficients) and
// the paper-only viscoelastic system.  Velocity at (i+1/2, j, k) etc.,
// normal stresses at nodes, shear stresses on edges (Virieux 1986):
//   D+ f(i) = sum_k c_k (f[i+k] - f[i-k+1])   (derivative at i+1/2)
//   D- f(i) = sum_k c_k (f[i+k-1] - f[i-k])   (derivative at i-1/2)
// Each phase reads its neighbours through L1/L2 (one thread per point,
// z-fastest warps -> coalesced rows).  Per-point arithmetic uses explicit
// _rn intrinsics so every launch geometry gives identical bits.
#include "common.cuh"

namespace sdmp {

struct ElParams {
  const float* __restrict__ in[16];
  float* __restrict__ out[12];
  Geom g;
  float c[3][SDMP_MAX_RADIUS];
  float dt;
};

template <int R>
__device__ __forceinline__ float dplus(const float* __restrict__ f, int64_t i, int64_t s,
                                       const float* c) {
  float acc = __fmul_rn(c[0], __fsub_rn(__ldg(f + i + s), __ldg(f + i)));
#pragma unroll
  for (int k = 2; k <= R; ++k)
    acc = __fmaf_rn(c[k - 1], __fsub_rn(__ldg(f + i + k * s), __ldg(f + i - (k - 1) * s)), acc);
  return acc;
}

template <int R>
__device__ __forceinline__ float dminus(const float* __restrict__ f, int64_t i, int64_t s,
                                        const float* c) {
  float acc = __fmul_rn(c[0], __fsub_rn(__ldg(f + i), __ldg(f + i - s)));
#pragma unroll
  for (int k = 2; k <= R; ++k)
    acc = __fmaf_rn(c[k - 1], __fsub_rn(__ldg(f + i + (k - 1) * s), __ldg(f + i - k * s)), acc);
  return acc;
}

#define EL_INDEX                                                               \
  const int z = p.g.lo[2] + blockIdx.x * 32 + threadIdx.x;                     \
  const int y = p.g.lo[1] + blockIdx.y * 8 + threadIdx.y;                      \
  const int x = p.g.lo[0] + blockIdx.z;                                        \
  if (z >= p.g.hi[2] || y >= p.g.hi[1]) return;                                \
  const int64_t sx = p.g.sx, sy = p.g.sy;                                      \
  const int64_t i = x * sx + y * sy + z;

// in = {vx, vy, vz, txx, tyy, tzz, txy, txz, tyz, b}; out = {vx1, vy1, vz1}
template <int R>
__global__ void __launch_bounds__(256) el_velocity(ElParams p) {
  EL_INDEX
  const float *txx = p.in[3], *tyy = p.in[4], *tzz = p.in[5];
  const float *txy = p.in[6], *txz = p.in[7], *tyz = p.in[8];
  float bdt = __fmul_rn(p.dt, __ldg(p.in[9] + i));
  float dvx = __fadd_rn(__fadd_rn(dplus<R>(txx, i, sx, p.c[0]), dminus<R>(txy, i, sy, p.c[1])),
                        dminus<R>(txz, i, 1, p.c[2]));
  float dvy = __fadd_rn(__fadd_rn(dminus<R>(txy, i, sx, p.c[0]), dplus<R>(tyy, i, sy, p.c[1])),
                        dminus<R>(tyz, i, 1, p.c[2]));
  float dvz = __fadd_rn(__fadd_rn(dminus<R>(txz, i, sx, p.c[0]), dminus<R>(tyz, i, sy, p.c[1])),
                        dplus<R>(tzz, i, 1, p.c[2]));
  p.out[0][i] = __fmaf_rn(bdt, dvx, __ldg(p.in[0] + i));
  p.out[1][i] = __fmaf_rn(bdt, dvy, __ldg(p.in[1] + i));
  p.out[2][i] = __fmaf_rn(bdt, dvz, __ldg(p.in[2] + i));
}

template <int R>
__device__ __forceinline__ void strains(const ElParams& p, int64_t i, int64_t sx, int64_t sy,
                                        float e[6]) {
  const float *vx = p.in[0], *vy = p.in[1], *vz = p.in[2];
  e[0] = dminus<R>(vx, i, sx, p.c[0]);
  e[1] = dminus<R>(vy, i, sy, p.c[1]);
  e[2] = dminus<R>(vz, i, 1, p.c[2]);
  e[3] = __fadd_rn(dplus<R>(vx, i, sy, p.c[1]), dplus<R>(vy, i, sx, p.c[0]));
  e[4] = __fadd_rn(dplus<R>(vx, i, 1, p.c[2]), dplus<R>(vz, i, sx, p.c[0]));
  e[5] = __fadd_rn(dplus<R>(vy, i, 1, p.c[2]), dplus<R>(vz, i, sy, p.c[1]));
}

// in = {vx1, vy1, vz1, txx..tyz (6), lam, mu}; out = {txx1..tyz1}
template <int R>
__global__ void __launch_bounds__(256) el_stress(ElParams p) {
  EL_INDEX
  float e[6];
  strains<R>(p, i, sx, sy, e);
  const float l = __ldg(p.in[9] + i), mu = __ldg(p.in[10] + i);
  const float tr = __fadd_rn(__fadd_rn(e[0], e[1]), e[2]);
  const float ltr = __fmul_rn(l, tr), m2 = __fmul_rn(2.f, mu);
#pragma unroll
  for (int c = 0; c < 3; ++c)
    p.out[c][i] = __fmaf_rn(p.dt, __fmaf_rn(m2, e[c], ltr), __ldg(p.in[3 + c] + i));
#pragma unroll
  for (int c = 3; c < 6; ++c)
    p.out[c][i] = __fmaf_rn(p.dt, __fmul_rn(mu, e[c]), __ldg(p.in[3 + c] + i));
}

// in = {vx1, vy1, vz1, s(6), r(6), l2m, mus, its} (18 > 16: params packed
// after r into in[15] region via out-of-line arrays below)
struct ViscoParams {
  ElParams e;
  const float* __restrict__ r0[6];
  const float* __restrict__ prm[3];
  float* __restrict__ r1[6];
};

template <int R>
__global__ void __launch_bounds__(256) visco_stress(ViscoParams vp) {
  const ElParams& p = vp.e;
  EL_INDEX
  float e[6];
  strains<R>(p, i, sx, sy, e);
  const float L = __ldg(vp.prm[0] + i), M = __ldg(vp.prm[1] + i), I = __ldg(vp.prm[2] + i);
  const float div = __fadd_rn(__fadd_rn(e[0], e[1]), e[2]);
  const float base = __fmul_rn(__fsub_rn(L, __fmul_rn(2.f, M)), div);
  const float m2 = __fmul_rn(2.f, M);
  const float dti = __fmul_rn(p.dt, I);
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    float A = c < 3 ? __fmaf_rn(m2, e[c], base) : __fmul_rn(M, e[c]);
    float r0v = __ldg(vp.r0[c] + i);
    float rn = __fmaf_rn(-dti, __fadd_rn(r0v, A), r0v);
    vp.r1[c][i] = rn;
    p.out[c][i] = __fmaf_rn(p.dt, __fadd_rn(A, rn), __ldg(p.in[3 + c] + i));
  }
}

static int fill(ElParams& p, const int64_t full[3], const int64_t lo[3], const int64_t hi[3],
                int radius, const float* sc, float dt) {
  int rc = make_geom(full, lo, hi, &p.g);
  if (rc) return rc;
  SDMP_CHECK(radius >= 1 && radius <= SDMP_MAX_RADIUS, "staggered radius outside 1..8");
  for (int a = 0; a < 3; ++a) {
    SDMP_CHECK(lo[a] >= radius && hi[a] + radius <= full[a], "box + radius exceeds FULL");
    for (int k = 0; k < SDMP_MAX_RADIUS; ++k)
      p.c[a][k] = k < radius ? sc[a * SDMP_MAX_RADIUS + k] : 0.f;
  }
  p.dt = dt;
  return SDMP_OK;
}

template <class P, class K>
static int launch(const Geom& g, K kernel, const P& params, cudaStream_t st) {
  dim3 b(32, 8);
  dim3 grid((g.hi[2] - g.lo[2] + 31) / 32, (g.hi[1] - g.lo[1] + 7) / 8, g.hi[0] - g.lo[0]);
  kernel<<<grid, b, 0, st>>>(params);
  SDMP_LAUNCHED();
  return SDMP_OK;
}

#define RADIUS_SWITCH(KERNEL, P)                                               \
  switch (radius) {                                                            \
    case 1: return launch(P.g, KERNEL<1>, params, st);                         \
    case 2: return launch(P.g, KERNEL<2>, params, st);                         \
    case 3: return launch(P.g, KERNEL<3>, params, st);                         \
    case 4: return launch(P.g, KERNEL<4>, params, st);                         \
    case 5: return launch(P.g, KERNEL<5>, params, st);                         \
    case 6: return launch(P.g, KERNEL<6>, params, st);                         \
    case 7: return launch(P.g, KERNEL<7>, params, st);                         \
    case 8: return launch(P.g, KERNEL<8>, params, st);                         \
  }                                                                            \
  set_error("unsupported radius");                                             \
  return SDMP_EUNSUPPORTED;

}  // namespace sdmp

using namespace sdmp;

extern "C" int sdmp_elastic_velocity(void* stream, const float* const v0[3],
                                     const float* const tau[6], const float* b,
                                     float* const v1[3], const int64_t full[3],
                                     const int64_t lo[3], const int64_t hi[3], int32_t radius,
                                     const float* sc, float dt) {
  ElParams params{};
  int rc = fill(params, full, lo, hi, radius, sc, dt);
  if (rc) return rc;
  if (box_empty(params.g)) return SDMP_OK;
  for (int c = 0; c < 3; ++c) params.in[c] = v0[c];
  for (int c = 0; c < 6; ++c) params.in[3 + c] = tau[c];
  params.in[9] = b;
  for (int c = 0; c < 3; ++c) params.out[c] = v1[c];
  cudaStream_t st = (cudaStream_t)stream;
  RADIUS_SWITCH(el_velocity, params)
}

extern "C" int sdmp_elastic_stress(void* stream, const float* const v1[3],
                                   const float* const t0[6], const float* lam, const float* mu,
                                   float* const t1[6], const int64_t full[3],
                                   const int64_t lo[3], const int64_t hi[3], int32_t radius,
                                   const float* sc, float dt) {
  ElParams params{};
  int rc = fill(params, full, lo, hi, radius, sc, dt);
  if (rc) return rc;
  if (box_empty(params.g)) return SDMP_OK;
  for (int c = 0; c < 3; ++c) params.in[c] = v1[c];
  for (int c = 0; c < 6; ++c) params.in[3 + c] = t0[c];
  params.in[9] = lam;
  params.in[10] = mu;
  for (int c = 0; c < 6; ++c) params.out[c] = t1[c];
  cudaStream_t st = (cudaStream_t)stream;
  RADIUS_SWITCH(el_stress, params)
}

extern "C" int sdmp_visco_stress(void* stream, const float* const v1[3],
                                 const float* const s0[6], const float* const r0[6],
                                 const float* const prm[3], float* const s1[6],
                                 float* const r1[6], const int64_t full[3], const int64_t lo[3],
                                 const int64_t hi[3], int32_t radius, const float* sc,
                                 float dt) {
  ViscoParams params{};
  int rc = fill(params.e, full, lo, hi, radius, sc, dt);
  if (rc) return rc;
  if (box_empty(params.e.g)) return SDMP_OK;
  for (int c = 0; c < 3; ++c) params.e.in[c] = v1[c];
  for (int c = 0; c < 6; ++c) {
    params.e.in[3 + c] = s0[c];
    params.e.out[c] = s1[c];
    params.r0[c] = r0[c];
    params.r1[c] = r1[c];
  }
  for (int c = 0; c < 3; ++c) params.prm[c] = prm[c];
  cudaStream_t st = (cudaStream_t)stream;
  RADIUS_SWITCH(visco_stress, params.e)
}
