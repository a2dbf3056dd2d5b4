// Sparse injection / interpolation and halo data
// movement (pack/unpack SPEC.md:430-438, box copies and completion flags
// for the NVLink peer exchange that replaces the SPEC Transport,
// SPEC.md:406-411) for sm_100a.
#include "common.cuh"

namespace sdmp {

// ---- sparse --------------------------------------------------------------

// One thread per owned grid node; contributions pre-sorted by point id on
// the host, summed sequentially: deterministic, no float atomics.
// `ctr` (plan mode): device step counter {time, steps}; the series row is
// ctr[0] - t0 (lets a captured CUDA graph replay across timesteps).
__global__ void k_inject(float* __restrict__ f, const int64_t* __restrict__ node,
                         const int32_t* __restrict__ ptr, int nnodes,
                         const int32_t* __restrict__ pid, const float* __restrict__ w,
                         const float* __restrict__ amps, float C, const float* __restrict__ m,
                         const int64_t* __restrict__ ctr, int64_t stride, int64_t t0,
                         const Push push) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= nnodes) return;
  if (ctr) amps += (ctr[0] - t0) * stride;
  float acc = 0.f;
  for (int j = ptr[n]; j < ptr[n + 1]; ++j) acc = __fmaf_rn(w[j], amps[pid[j]], acc);
  const int64_t i = node[n];
  const float s = m ? __fdiv_rn(C, m[i]) : C;
  const float v = __fmaf_rn(acc, s, f[i]);
  f[i] = v;
  if (push.ndir) {  // full mode: the injected value also reaches the peers' halos
    const int x = (int)(i / push.msx);
    const int64_t rem = i - (int64_t)x * push.msx;
    const int y = (int)(rem / push.msy);
    const int z = (int)(rem - (int64_t)y * push.msy);
    push_point(push, x, y, z, &v, 1);
  }
}

__global__ void k_interp(const float* __restrict__ f, const int64_t* __restrict__ idx,
                         const float* __restrict__ w, int npts, int nc, float* __restrict__ out,
                         const int64_t* __restrict__ ctr, int64_t stride, int64_t t0) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= npts) return;
  if (ctr) out += (ctr[0] - t0) * stride;
  float acc = 0.f;
  for (int c = 0; c < nc; ++c) acc = __fmaf_rn(w[p * nc + c], __ldg(f + idx[p * nc + c]), acc);
  out[p] = acc;
}

int inject(cudaStream_t st, float* field, const int64_t* node, const int32_t* ptr, int nnodes,
           const int32_t* pid, const float* w, const float* amps, float C, const float* m,
           const int64_t* ctr, int64_t stride, int64_t t0, const Push* push) {
  if (nnodes <= 0) return SDMP_OK;
  SDMP_CHECK(field && node && ptr && pid && w && amps, "inject: null array");
  const Push nopush{};
  k_inject<<<(nnodes + 127) / 128, 128, 0, st>>>(field, node, ptr, nnodes, pid, w, amps, C, m,
                                                 ctr, stride, t0, push ? *push : nopush);
  SDMP_LAUNCHED();
  return SDMP_OK;
}

int interpolate(cudaStream_t st, const float* field, const int64_t* idx, const float* w,
                int npts, int nc, float* out, const int64_t* ctr, int64_t stride, int64_t t0) {
  if (npts <= 0) return SDMP_OK;
  SDMP_CHECK(field && idx && w && out, "interpolate: null array");
  k_interp<<<(npts + 127) / 128, 128, 0, st>>>(field, idx, w, npts, nc, out, ctr, stride, t0);
  SDMP_LAUNCHED();
  return SDMP_OK;
}

// ---- parameter binding --------------------------------------------------

__global__ void k_bind_scale(float* __restrict__ out, const float* __restrict__ in, int64_t n,
                             float C) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float v = in[i];
    out[i] = v != 0.f ? __fdiv_rn(C, v) : 0.f;
  }
}

int bind_scale(cudaStream_t st, float* out, const float* in, int64_t n, float C) {
  if (n <= 0) return SDMP_OK;
  SDMP_CHECK(out && in, "bind_scale: null array");
  int64_t blocks = (n + 255) / 256;
  if (blocks > 8 * 148 * 8) blocks = 8 * 148 * 8;
  k_bind_scale<<<(unsigned)blocks, 256, 0, st>>>(out, in, n, C);
  SDMP_LAUNCHED();
  return SDMP_OK;
}

// ---- pack / unpack / box copy ---------------------------------------------

struct BoxXfer {
  const float* __restrict__ src;
  float* __restrict__ dst;
  int64_t ssx, ssy, dsx, dsy;  // strides (z stride 1)
  int64_t soff, doff;          // element offset of the box origin
  int ex, ey, ez;              // extent
};

// grid: x = z-chunks, y = y rows, z = x planes
__global__ void k_box_copy(BoxXfer b) {
  const int y = blockIdx.y, x = blockIdx.z;
  const float* s = b.src + b.soff + x * b.ssx + y * b.ssy;
  float* d = b.dst + b.doff + x * b.dsx + y * b.dsy;
  for (int z = blockIdx.x * blockDim.x + threadIdx.x; z < b.ez; z += gridDim.x * blockDim.x)
    d[z] = s[z];
}

static int box_copy_kernel(cudaStream_t st, const BoxXfer& b) {
  if (b.ex <= 0 || b.ey <= 0 || b.ez <= 0) return SDMP_OK;
  SDMP_CHECK(b.ey <= 65535 && b.ex <= 65535, "box copy extent too large");
  int zb = (b.ez + 255) / 256;
  if (zb > 8) zb = 8;
  dim3 grid(zb, b.ey, b.ex);
  k_box_copy<<<grid, 256, 0, st>>>(b);
  SDMP_LAUNCHED();
  return SDMP_OK;
}

// ---- batched halo copy: every message of one post in ONE kernel ------------
// (diagonal / basic mode with SDMP_COPY_ENGINE=batch).  Rows (x, y) of all
// boxes are flattened; each warp moves one z row per iteration with 16-byte
// loads / peer stores when the row is 16-byte aligned on both sides (the
// whole-z rows of the product always are), scalar otherwise.

__global__ void __launch_bounds__(256) k_multi_copy(const __grid_constant__ MultiCopy mc) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < mc.rows;
       r += nwarps) {
    int m = 0;
    while (m + 1 < mc.n && mc.row0[m + 1] <= r) ++m;
    const CopyMsg& c = mc.m[m];
    const int64_t rr = r - mc.row0[m];
    const int64_t x = rr / c.ey, y = rr - x * c.ey;
    const float* s = c.src + c.soff + x * c.ssx + y * c.ssy;
    float* d = c.dst + c.doff + x * c.dsx + y * c.dsy;
    const int ez = c.ez;
    if (((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d)) & 15) == 0) {
      const int n4 = ez >> 2;
      const float4* s4 = reinterpret_cast<const float4*>(s);
      float4* d4 = reinterpret_cast<float4*>(d);
      for (int i = lane; i < n4; i += 32) d4[i] = __ldg(s4 + i);
      for (int i = (n4 << 2) + lane; i < ez; i += 32) d[i] = s[i];
    } else {
      for (int i = lane; i < ez; i += 32) d[i] = s[i];
    }
  }
}

int multi_copy(cudaStream_t st, const MultiCopy& mc) {
  if (mc.n <= 0 || mc.rows <= 0) return SDMP_OK;
  int64_t blocks = (mc.rows + 7) / 8;
  const int64_t cap = 2ll * num_sms();
  if (blocks > cap) blocks = cap;
  k_multi_copy<<<(unsigned)blocks, 256, 0, st>>>(mc);
  SDMP_LAUNCHED();
  return SDMP_OK;
}

int pack(cudaStream_t st, const float* field, const int64_t full[3], const int64_t lo[3],
         const int64_t hi[3], float* buf) {
  Geom g;
  int rc = make_geom(full, lo, hi, &g);
  if (rc) return rc;
  BoxXfer b{};
  b.src = field; b.dst = buf;
  b.ssx = g.sx; b.ssy = g.sy;
  b.ex = g.hi[0] - g.lo[0]; b.ey = g.hi[1] - g.lo[1]; b.ez = g.hi[2] - g.lo[2];
  b.dsy = b.ez; b.dsx = (int64_t)b.ey * b.ez;
  b.soff = g.lo[0] * g.sx + g.lo[1] * g.sy + g.lo[2];
  b.doff = 0;
  return box_copy_kernel(st, b);
}

int unpack(cudaStream_t st, float* field, const int64_t full[3], const int64_t lo[3],
           const int64_t hi[3], const float* buf) {
  Geom g;
  int rc = make_geom(full, lo, hi, &g);
  if (rc) return rc;
  BoxXfer b{};
  b.src = buf; b.dst = field;
  b.dsx = g.sx; b.dsy = g.sy;
  b.ex = g.hi[0] - g.lo[0]; b.ey = g.hi[1] - g.lo[1]; b.ez = g.hi[2] - g.lo[2];
  b.ssy = b.ez; b.ssx = (int64_t)b.ey * b.ez;
  b.doff = g.lo[0] * g.sx + g.lo[1] * g.sy + g.lo[2];
  b.soff = 0;
  return box_copy_kernel(st, b);
}

int copy_box(cudaStream_t st, const float* src, const int64_t sfull[3], const int64_t slo[3],
             float* dst, const int64_t dfull[3], const int64_t dlo[3], const int64_t ext[3],
             int engine) {
  for (int a = 0; a < 3; ++a) {
    SDMP_CHECK(ext[a] >= 0, "negative extent");
    SDMP_CHECK(slo[a] >= 0 && slo[a] + ext[a] <= sfull[a], "source box outside array");
    SDMP_CHECK(dlo[a] >= 0 && dlo[a] + ext[a] <= dfull[a], "destination box outside array");
  }
  if (ext[0] == 0 || ext[1] == 0 || ext[2] == 0) return SDMP_OK;
  if (engine == 2) {  // the batched post kernel (k_multi_copy) with one box
    MultiCopy mc;
    CopyMsg& c = mc.m[0];
    c.src = src; c.dst = dst;
    c.ssy = sfull[2]; c.ssx = sfull[1] * sfull[2];
    c.dsy = dfull[2]; c.dsx = dfull[1] * dfull[2];
    c.soff = slo[0] * c.ssx + slo[1] * c.ssy + slo[2];
    c.doff = dlo[0] * c.dsx + dlo[1] * c.dsy + dlo[2];
    c.ex = (int)ext[0]; c.ey = (int)ext[1]; c.ez = (int)ext[2];
    mc.n = 1;
    mc.row0[0] = 0;
    mc.rows = (int64_t)c.ex * c.ey;
    return multi_copy(st, mc);
  }
  if (engine == 0) {
    cudaMemcpy3DParms p = {};
    p.srcPtr = make_cudaPitchedPtr((void*)src, sfull[2] * sizeof(float), sfull[2], sfull[1]);
    p.dstPtr = make_cudaPitchedPtr(dst, dfull[2] * sizeof(float), dfull[2], dfull[1]);
    p.srcPos = make_cudaPos(slo[2] * sizeof(float), slo[1], slo[0]);
    p.dstPos = make_cudaPos(dlo[2] * sizeof(float), dlo[1], dlo[0]);
    p.extent = make_cudaExtent(ext[2] * sizeof(float), ext[1], ext[0]);
    p.kind = cudaMemcpyDefault;
    SDMP_CUDA(cudaMemcpy3DAsync(&p, st));
    return SDMP_OK;
  }
  BoxXfer b{};
  b.src = src; b.dst = dst;
  b.ssy = sfull[2]; b.ssx = sfull[1] * sfull[2];
  b.dsy = dfull[2]; b.dsx = dfull[1] * dfull[2];
  b.soff = slo[0] * b.ssx + slo[1] * b.ssy + slo[2];
  b.doff = dlo[0] * b.dsx + dlo[1] * b.dsy + dlo[2];
  b.ex = (int)ext[0]; b.ey = (int)ext[1]; b.ez = (int)ext[2];
  return box_copy_kernel(st, b);
}

// ---- completion flags ------------------------------------------------------

struct FlagArgs {
  uint32_t* ptr[32];
  int n;
  uint32_t value;
  unsigned long long timeout_ns;
  int* err;             // host-mapped watchdog word
  const int64_t* ctr;   // plan mode: epoch = ctr[1] * phases + phase + 1
  int phases, phase;
};

__device__ __forceinline__ uint32_t flag_value(const FlagArgs& a) {
  return a.ctr ? (uint32_t)(a.ctr[1] * a.phases + a.phase + 1) : a.value;
}

// Writes `value` into each (peer) flag with system-scope release semantics,
// after all prior work on the stream (copies into the peer's halo).
__global__ void k_signal(FlagArgs a) {
  const int i = threadIdx.x;
  if (i >= a.n) return;
  const uint32_t value = flag_value(a);
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.ptr[i]), "r"(value) : "memory");
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Spins (with backoff) until every flag >= value (wrap-safe), or the
// watchdog expires: then records the failure and returns so the stream
// never hangs (SPEC.md:468 watchdog).
__global__ void k_wait(FlagArgs a) {
  const int i = threadIdx.x;
  if (i >= a.n) return;
  const uint32_t value = flag_value(a);
  const unsigned long long t0 = gtimer();
  while (true) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(a.ptr[i]) : "memory");
    if ((int32_t)(v - value) >= 0) break;
    if (gtimer() - t0 > a.timeout_ns) {
      atomicExch(a.err, 1);
      break;
    }
    __nanosleep(200);
  }
}

int signal_flags(cudaStream_t st, uint32_t* const* ptrs, int n, uint32_t value,
                 const int64_t* ctr, int phases, int phase) {
  if (n <= 0) return SDMP_OK;
  SDMP_CHECK(n <= 32, "at most 32 flags per signal");
  FlagArgs a{};
  for (int i = 0; i < n; ++i) a.ptr[i] = ptrs[i];
  a.n = n;
  a.value = value;
  a.ctr = ctr;
  a.phases = phases;
  a.phase = phase;
  k_signal<<<1, 32, 0, st>>>(a);
  SDMP_LAUNCHED();
  return SDMP_OK;
}

int wait_flags(cudaStream_t st, uint32_t* const* ptrs, int n, uint32_t value,
               unsigned long long timeout_ns, int* err, const int64_t* ctr, int phases,
               int phase) {
  if (n <= 0) return SDMP_OK;
  SDMP_CHECK(n <= 32, "at most 32 flags per wait");
  FlagArgs a{};
  for (int i = 0; i < n; ++i) a.ptr[i] = ptrs[i];
  a.n = n;
  a.value = value;
  a.timeout_ns = timeout_ns;
  a.err = err;
  a.ctr = ctr;
  a.phases = phases;
  a.phase = phase;
  k_wait<<<1, 32, 0, st>>>(a);
  SDMP_LAUNCHED();
  return SDMP_OK;
}

// ---- plan step counter -------------------------------------------------------

__global__ void k_set_ctr(int64_t* ctr, int64_t time, int64_t steps) {
  ctr[0] = time;
  ctr[1] = steps;
}

__global__ void k_tick(int64_t* ctr) {
  ctr[0] += 1;
  ctr[1] += 1;
}

int set_ctr(cudaStream_t st, int64_t* ctr, int64_t time, int64_t steps) {
  k_set_ctr<<<1, 1, 0, st>>>(ctr, time, steps);
  SDMP_LAUNCHED();
  return SDMP_OK;
}

int tick_ctr(cudaStream_t st, int64_t* ctr) {
  k_tick<<<1, 1, 0, st>>>(ctr);
  SDMP_LAUNCHED();
  return SDMP_OK;
}

}  // namespace sdmp

using namespace sdmp;

extern "C" int sdmp_inject(void* stream, float* field, const int64_t* node, const int32_t* ptr,
                           int32_t nnodes, const int32_t* pid, const float* w,
                           const float* amps, float C, const float* m) {
  return inject((cudaStream_t)stream, field, node, ptr, nnodes, pid, w, amps, C, m, nullptr, 0,
                0, nullptr);
}

extern "C" int sdmp_interpolate(void* stream, const float* field, const int64_t* idx,
                                const float* w, int32_t npts, int32_t ncorner, float* out) {
  return interpolate((cudaStream_t)stream, field, idx, w, npts, ncorner, out, nullptr, 0, 0);
}

extern "C" int sdmp_bind_scale(void* stream, float* out, const float* in, int64_t n, float C) {
  return bind_scale((cudaStream_t)stream, out, in, n, C);
}

extern "C" int sdmp_pack(void* stream, const float* field, const int64_t full[3],
                         const int64_t lo[3], const int64_t hi[3], float* buf) {
  return pack((cudaStream_t)stream, field, full, lo, hi, buf);
}

extern "C" int sdmp_unpack(void* stream, float* field, const int64_t full[3],
                           const int64_t lo[3], const int64_t hi[3], const float* buf) {
  return unpack((cudaStream_t)stream, field, full, lo, hi, buf);
}

extern "C" int sdmp_copy_box(void* stream, const float* src, const int64_t src_full[3],
                             const int64_t src_lo[3], float* dst, const int64_t dst_full[3],
                             const int64_t dst_lo[3], const int64_t extent[3], int32_t engine) {
  return copy_box((cudaStream_t)stream, src, src_full, src_lo, dst, dst_full, dst_lo, extent,
                  engine);
}
