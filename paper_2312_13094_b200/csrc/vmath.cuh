// Value-type arithmetic for the shared per-point routines.
//
// Every stencil family evaluates a point with ONE templated routine whose
// value type is `float` (generic one-thread-per-point kernels) or `V2` (two
// consecutive z points per thread in the TMA stream engine, mapped onto
// Blackwell's packed fp32 instructions FFMA2 / FADD2 / FMUL2).  Each lane of
// a V2 operation performs exactly the scalar round-to-nearest operation, so
// both launch shapes produce identical bits — PROVIDED no separately rounded
// product feeds an add (ptxas contracts packed mul.rn + add.rn into FFMA2).
// The routines therefore only use forms ptxas cannot contract differently:
// products feed fma multiplicands / addends of an fma, or are written as
// explicit fma.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace sdmp {

struct V2 {
  uint64_t r;  // packed {lo = z, hi = z + 1}
};

__device__ __forceinline__ V2 v2pack(float a, float b) {
  V2 o;
  asm("mov.b64 %0, {%1, %2};" : "=l"(o.r) : "f"(a), "f"(b));
  return o;
}
__device__ __forceinline__ float v2lo(V2 v) {
  float a;
  asm("mov.b64 {%0, _}, %1;" : "=f"(a) : "l"(v.r));
  return a;
}
__device__ __forceinline__ float v2hi(V2 v) {
  float b;
  asm("mov.b64 {_, %0}, %1;" : "=f"(b) : "l"(v.r));
  return b;
}
__device__ __forceinline__ V2 v2bcast(float a) { return v2pack(a, a); }

// ---- float ----------------------------------------------------------------
__device__ __forceinline__ float vadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float vsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float vmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float vfma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ float vneg(float a) { return -a; }
// 0 - a (exact negation up to the sign of zero): one FADD2 / folded into a
// packed operand's negate modifier, where vneg costs two LOP3 per pair
__device__ __forceinline__ float vnegz(float a) { return __fsub_rn(0.f, a); }
// -(a b) rounded once, as 0 - RN(a b): ptxas emits FFMA2 -a, b, 0 for pairs
__device__ __forceinline__ float vnmul(float a, float b) { return __fsub_rn(0.f, __fmul_rn(a, b)); }
__device__ __forceinline__ float vdiv(float a, float b) { return __fdiv_rn(a, b); }
// coefficient (uniform scalar) times value
__device__ __forceinline__ float vcmul(float c, float b) { return __fmul_rn(c, b); }
__device__ __forceinline__ float vcfma(float c, float b, float acc) { return __fmaf_rn(c, b, acc); }
template <class T> __device__ __forceinline__ T vconst(float c);
template <> __device__ __forceinline__ float vconst<float>(float c) { return c; }

// ---- V2 (packed fp32x2) ---------------------------------------------------------
__device__ __forceinline__ V2 vadd(V2 a, V2 b) {
  V2 o;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(o.r) : "l"(a.r), "l"(b.r));
  return o;
}
__device__ __forceinline__ V2 vsub(V2 a, V2 b) {
  V2 o;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(o.r) : "l"(a.r), "l"(b.r));
  return o;
}
__device__ __forceinline__ V2 vmul(V2 a, V2 b) {
  V2 o;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(o.r) : "l"(a.r), "l"(b.r));
  return o;
}
__device__ __forceinline__ V2 vfma(V2 a, V2 b, V2 c) {
  V2 o;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(o.r) : "l"(a.r), "l"(b.r), "l"(c.r));
  return o;
}
__device__ __forceinline__ V2 vnegz(V2 a) { return vsub(v2bcast(0.f), a); }
__device__ __forceinline__ V2 vnmul(V2 a, V2 b) { return vsub(v2bcast(0.f), vmul(a, b)); }
__device__ __forceinline__ V2 vneg(V2 a) {
  // sign flip of both lanes (exact)
  V2 o;
  o.r = a.r ^ 0x8000000080000000ull;
  return o;
}
__device__ __forceinline__ V2 vdiv(V2 a, V2 b) {
  return v2pack(__fdiv_rn(v2lo(a), v2lo(b)), __fdiv_rn(v2hi(a), v2hi(b)));
}
__device__ __forceinline__ V2 vcmul(float c, V2 b) { return vmul(v2bcast(c), b); }
__device__ __forceinline__ V2 vcfma(float c, V2 b, V2 acc) { return vfma(v2bcast(c), b, acc); }
template <> __device__ __forceinline__ V2 vconst<V2>(float c) { return v2bcast(c); }

}  // namespace sdmp
