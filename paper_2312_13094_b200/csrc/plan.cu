// Plan executor, library entry points and inter-process memory for libsdmp.
//
// The host planner (paper_2312_13094_b200/compiler.py) lowers an Operator to
// an ExecPlan: an ordered list of per-timestep
// actions — compute(box, kernel), exchange post / wait, sparse inject /
// interpolate, stream joins.  This file replays that list for
// time_m..time_M on three CUDA streams:
//   0  compute (CORE / DOMAIN),
//   1  remainder (OWNED slabs; highest priority),
//   2  exchange (copy-engine / peer-store halo pushes + completion flags).
// Halo exchange is a PUSH over NVLink: a rank copies its OWNED boundary
// boxes straight into the neighbour's HALO (IPC-mapped pointers; no pack /
// unpack), then releases a per-direction flag in the neighbour's memory with
// the phase epoch; the neighbour's WAIT acquires it on the device.  This
// realises execute_plan_full and halo_exchange
// basic/diagonal without host round trips.
#include <cuda.h>

#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace sdmp {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
const char* get_error() { return g_err.c_str(); }

int star_update(cudaStream_t, const float*, const float*, const float*, float*, const int64_t*,
                const int64_t*, const int64_t*, const int32_t*, const float*, float, float, float,
                int, const Push*);
int var_star_update(cudaStream_t, const float*, const float*, const float*, const float*,
                    const float*, float*, const int64_t*, const int64_t*, const int64_t*,
                    const int32_t*, const float*, int, const Push*);
int rot_update_entry(cudaStream_t, const float* const*, float*, const int64_t*, const int64_t*,
                     const int64_t*, int32_t, const float*, float, const Push*);
int tti_update_entry(cudaStream_t, const float* const*, float*, float*, const int64_t*,
                     const int64_t*, const int64_t*, int32_t, const float*, const float*, float,
                     const Push*);
int inject(cudaStream_t, float*, const int64_t*, const int32_t*, int, const int32_t*,
           const float*, const float*, float, const float*, const int64_t*, int64_t, int64_t,
           const Push*);
int elastic_velocity_impl(void*, const float* const[3], const float* const[6], const float*,
                          float* const[3], const int64_t[3], const int64_t[3], const int64_t[3],
                          int32_t, const float*, float, const Push*, bool);
int elastic_stress_impl(void*, const float* const[3], const float* const[6], const float*,
                        const float*, float* const[6], const int64_t[3], const int64_t[3],
                        const int64_t[3], int32_t, const float*, float, const Push*, bool);
int visco_stress_impl(void*, const float* const[3], const float* const[6],
                      const float* const[6], const float* const[3], float* const[6],
                      float* const[6], const int64_t[3], const int64_t[3], const int64_t[3],
                      int32_t, const float*, float, const Push*);
int interpolate(cudaStream_t, const float*, const int64_t*, const float*, int, int, float*,
                const int64_t*, int64_t, int64_t);
int set_ctr(cudaStream_t, int64_t*, int64_t, int64_t);
int tick_ctr(cudaStream_t, int64_t*);
int copy_box(cudaStream_t, const float*, const int64_t*, const int64_t*, float*, const int64_t*,
             const int64_t*, const int64_t*, int);
int signal_flags(cudaStream_t, uint32_t* const*, int, uint32_t, const int64_t*, int, int);
int wait_flags(cudaStream_t, uint32_t* const*, int, uint32_t, unsigned long long, int*,
               const int64_t*, int, int);

}  // namespace sdmp

using namespace sdmp;

namespace {

struct Field {
  int nbuf;
  uint64_t ptr[8];
  int64_t full[3];
};

struct SparseSet {
  int kind;  // 0 inject, 1 interpolate
  int npts, nnodes, ncorner;
  const int64_t* node;
  const int32_t* ptr;
  const int32_t* pid;
  const float* w;
  float* series;  // inject: amps[nt * npts]; interpolate: traces[nt * npts]
  int64_t stride, t0;
};

struct Action {
  std::vector<int64_t> i;
  std::vector<float> f;
};

}  // namespace

struct sdmp_plan {
  int device = 0;
  int phases = 1;
  cudaStream_t s[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t ev_step = nullptr, ev_join[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t ev_user[32];
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  // copy-engine fan-out for halo posts: messages round-robin over kCopy
  // streams so several copy engines move faces/edges concurrently
#ifndef SDMP_COPY_STREAMS
#define SDMP_COPY_STREAMS 4
#endif
  static constexpr int kCopy = SDMP_COPY_STREAMS;
  cudaStream_t cs[kCopy] = {};
  cudaEvent_t ev_fork = nullptr, ev_cdone[kCopy] = {};
  std::vector<Field> fields;
  std::vector<uint32_t*> flags;  // peer flag arrays
  uint32_t* local_flags = nullptr;
  std::vector<SparseSet> sparse;
  std::vector<Action> actions;
  int64_t steps_done = 0;
  int64_t run_time_m = 0;  // first timestep of the current run
  // device step counter {time, steps_done}: sparse rows and exchange epochs
  // are read from it so a captured period of steps can be replayed
  int64_t* dev_ctr = nullptr;
  bool graph_on = false;
  int period = 1;
  std::map<int64_t, cudaGraphExec_t> graphs;  // by time % period
  int* err_host = nullptr;
  int* err_dev = nullptr;
  int64_t timeout_ms = 30000;
  bool tracing = false;
  std::vector<cudaEvent_t> tr_beg, tr_end;
  cudaEvent_t tr_origin = nullptr;
  int last_traced = 0;
};

namespace {

float* resolve(const sdmp_plan* p, int64_t f, int64_t t, int64_t time) {
  if (f < 0) return nullptr;
  const Field& fl = p->fields[f];
  int64_t b = ((time + t) % fl.nbuf + fl.nbuf) % fl.nbuf;
  return reinterpret_cast<float*>(fl.ptr[b]);
}

// Optional fused-push block appended to a compute / inject action:
// [kPushMagic, ndir, nout, tshift, ndir x (lo3, hi3, off3), nout x ndir peer
// field ids (output-major)].  Peer buffers are resolved for this timestep.
constexpr int64_t kPushMagic = -77;

int base_len(int kind) {
  switch (kind) {
    case SDMP_ACT_STAR: return 19;
    case SDMP_ACT_VSTAR: return 21;
    case SDMP_ACT_ROT: return 23;
    case SDMP_ACT_TTI: return 33;
    case SDMP_ACT_EL_V: return 35;
    case SDMP_ACT_EL_T: return 43;
    case SDMP_ACT_VISCO_T: return 69;
    case SDMP_ACT_INJECT: return 6;
    default: return -1;
  }
}

// returns 1 if a push block was decoded into *out, 0 if none, < 0 on error
int parse_push(const sdmp_plan* p, const Action& a, int64_t time, Push* out) {
  const int b = base_len((int)a.i[0]);
  if (b < 0 || (int64_t)a.i.size() <= b || a.i[b] != kPushMagic) return 0;
  const int64_t* I = a.i.data() + b;
  const int ndir = (int)I[1], nout = (int)I[2];
  const int64_t tsh = I[3];
  SDMP_CHECK(ndir >= 0 && ndir <= kPushDirs && nout >= 1 && nout <= kPushOut, "push sizes");
  SDMP_CHECK((int64_t)a.i.size() >= b + 4 + 9 * ndir + nout * ndir, "push block truncated");
  out->ndir = ndir;
  out->nout = nout;
  const int64_t* gp = I + 4;
  const int64_t* fid = I + 4 + 9 * ndir;
  for (int d = 0; d < ndir; ++d) {
    PushGeo& g = out->geo[d];
    for (int k = 0; k < 3; ++k) {
      g.lo[k] = (int)gp[9 * d + k];
      g.hi[k] = (int)gp[9 * d + 3 + k];
      g.off[k] = (int)gp[9 * d + 6 + k];
    }
    // field id -1: the neighbour never reads output q across this face
    // (per-field halo radii, compiler.HaloSpot.sends); the kernels skip a
    // null base.  Strides come from the first output that is sent.
    int64_t pf = -1;
    for (int q = 0; q < nout; ++q) {
      const int64_t f = fid[q * ndir + d];
      SDMP_CHECK(f >= -1 && f < (int64_t)p->fields.size(), "push field id");
      out->base[q][d] = f >= 0 ? resolve(p, f, tsh, time) : nullptr;
      if (pf < 0) pf = f;
    }
    SDMP_CHECK(pf >= 0, "push direction without any field");
    g.psy = p->fields[pf].full[2];
    g.psx = p->fields[pf].full[1] * p->fields[pf].full[2];
  }
  const int64_t lf = a.i[2];  // first field of the action: this rank's layout
  out->msy = p->fields[lf].full[2];
  out->msx = p->fields[lf].full[1] * p->fields[lf].full[2];
  return 1;
}

// Kernel launches one action issues per step (copy-engine copies are not
// kernel launches).
int launches_of(const Action& a) {
  switch ((int)a.i[0]) {
    case SDMP_ACT_STAR: case SDMP_ACT_VSTAR: case SDMP_ACT_EL_V: case SDMP_ACT_EL_T:
    case SDMP_ACT_VISCO_T: case SDMP_ACT_INJECT: case SDMP_ACT_INTERP: case SDMP_ACT_WAIT:
      return 1;
    case SDMP_ACT_TTI: case SDMP_ACT_ROT:
      return 2;
    case SDMP_ACT_POST:
      return 1 + (a.i[4] == 1 ? (int)a.i[3] : 0);
    default:
      return 0;
  }
}

int run_action(sdmp_plan* p, const Action& a, int64_t time) {
  const int64_t* I = a.i.data();
  const float* F = a.f.data();
  const int kind = (int)I[0];
  cudaStream_t st = p->s[I[1]];
  Push push;
  const int hp = parse_push(p, a, time, &push);
  if (hp < 0) return hp;
  const Push* pp = hp ? &push : nullptr;
  switch (kind) {
    case SDMP_ACT_STAR: {
      // [k,s, fu0,tu0, fu2,tu2, fm, fu1,tu1, lo3, hi3, r3, variant]
      const float* u0 = resolve(p, I[2], I[3], time);
      const float* u2 = resolve(p, I[4], I[5], time);
      const float* m = resolve(p, I[6], 0, time);
      float* u1 = resolve(p, I[7], I[8], time);
      const int64_t* lo = I + 9;
      const int64_t* hi = I + 12;
      int32_t r[3] = {(int32_t)I[15], (int32_t)I[16], (int32_t)I[17]};
      const int nc = 3 * SDMP_NCOEF;
      return star_update(st, u0, u2, m, u1, p->fields[I[2]].full, lo, hi, r, F, F[nc],
                         F[nc + 1], F[nc + 2], (int)I[18], pp);
    }
    case SDMP_ACT_VSTAR: {
      // [k,s, fu0,tu0, fu2,tu2, fA, fB, fS, fu1,tu1, lo3, hi3, r3, variant]
      const float* u0 = resolve(p, I[2], I[3], time);
      const float* u2 = resolve(p, I[4], I[5], time);
      const float* A = resolve(p, I[6], 0, time);
      const float* B = resolve(p, I[7], 0, time);
      const float* Sv = resolve(p, I[8], 0, time);
      float* u1 = resolve(p, I[9], I[10], time);
      int32_t r[3] = {(int32_t)I[17], (int32_t)I[18], (int32_t)I[19]};
      return var_star_update(st, u0, u2, A, B, Sv, u1, p->fields[I[2]].full, I + 11, I + 14, r,
                             F, (int)I[20], pp);
    }
    case SDMP_ACT_ROT: {
      // [k,s, (fid,t) x {u0, u2, m, ax, ay, az}, fu1,tu1, lo3, hi3, R]
      const float* in[6];
      for (int k = 0; k < 6; ++k) in[k] = resolve(p, I[2 + 2 * k], I[3 + 2 * k], time);
      float* u1 = resolve(p, I[14], I[15], time);
      const int nc = 3 * SDMP_NCOEF;
      return rot_update_entry(st, in, u1, p->fields[I[2]].full, I + 16, I + 19, (int32_t)I[22],
                              F, F[nc], pp);
    }
    case SDMP_ACT_TTI: {
      const float* in[10];
      for (int k = 0; k < 10; ++k) in[k] = resolve(p, I[2 + 2 * k], I[3 + 2 * k], time);
      float* p1 = resolve(p, I[22], I[23], time);
      float* r1 = resolve(p, I[24], I[25], time);
      const int64_t* lo = I + 26;
      const int64_t* hi = I + 29;
      const int nc = 3 * SDMP_NCOEF;
      return tti_update_entry(st, in, p1, r1, p->fields[I[2]].full, lo, hi, (int32_t)I[32], F,
                              F + nc, F[2 * nc], pp);
    }
    case SDMP_ACT_EL_V: {
      const float* v0[3]; const float* tau[6]; float* v1[3];
      for (int k = 0; k < 3; ++k) v0[k] = resolve(p, I[2 + 2 * k], I[3 + 2 * k], time);
      for (int k = 0; k < 6; ++k) tau[k] = resolve(p, I[8 + 2 * k], I[9 + 2 * k], time);
      const float* b = resolve(p, I[20], I[21], time);
      for (int k = 0; k < 3; ++k) v1[k] = resolve(p, I[22 + 2 * k], I[23 + 2 * k], time);
      const int64_t* lo = I + 28;
      const int64_t* hi = I + 31;
      // radius | collocated << 8 (the SPEC's collocated elastic_kernel)
      return elastic_velocity_impl(st, v0, tau, b, v1, p->fields[I[2]].full, lo, hi,
                                   (int32_t)(I[34] & 0xff), F, F[3 * SDMP_MAX_RADIUS], pp,
                                   (I[34] >> 8) & 1);
    }
    case SDMP_ACT_EL_T: {
      const float* v1[3]; const float* t0[6]; float* t1[6];
      for (int k = 0; k < 3; ++k) v1[k] = resolve(p, I[2 + 2 * k], I[3 + 2 * k], time);
      for (int k = 0; k < 6; ++k) t0[k] = resolve(p, I[8 + 2 * k], I[9 + 2 * k], time);
      const float* lam = resolve(p, I[20], I[21], time);
      const float* mu = resolve(p, I[22], I[23], time);
      for (int k = 0; k < 6; ++k) t1[k] = resolve(p, I[24 + 2 * k], I[25 + 2 * k], time);
      const int64_t* lo = I + 36;
      const int64_t* hi = I + 39;
      return elastic_stress_impl(st, v1, t0, lam, mu, t1, p->fields[I[2]].full, lo, hi,
                                 (int32_t)(I[42] & 0xff), F, F[3 * SDMP_MAX_RADIUS], pp,
                                 (I[42] >> 8) & 1);
    }
    case SDMP_ACT_VISCO_T: {
      const float* v1[3]; const float* s0[6]; const float* r0[6]; const float* prm[3];
      float* s1[6]; float* r1[6];
      int o = 2;
      for (int k = 0; k < 3; ++k, o += 2) v1[k] = resolve(p, I[o], I[o + 1], time);
      for (int k = 0; k < 6; ++k, o += 2) s0[k] = resolve(p, I[o], I[o + 1], time);
      for (int k = 0; k < 6; ++k, o += 2) r0[k] = resolve(p, I[o], I[o + 1], time);
      for (int k = 0; k < 3; ++k, o += 2) prm[k] = resolve(p, I[o], I[o + 1], time);
      for (int k = 0; k < 6; ++k, o += 2) s1[k] = resolve(p, I[o], I[o + 1], time);
      for (int k = 0; k < 6; ++k, o += 2) r1[k] = resolve(p, I[o], I[o + 1], time);
      const int64_t* lo = I + o;
      const int64_t* hi = I + o + 3;
      return visco_stress_impl(st, v1, s0, r0, prm, s1, r1, p->fields[I[2]].full, lo, hi,
                               (int32_t)I[o + 6], F, F[3 * SDMP_MAX_RADIUS], pp);
    }
    case SDMP_ACT_INJECT: {
      // [k,s, ffield,t, fm, set]
      float* fld = resolve(p, I[2], I[3], time);
      const float* m = resolve(p, I[4], 0, time);
      const SparseSet& ss = p->sparse[I[5]];
      if (time < ss.t0) return SDMP_OK;
      return inject(st, fld, ss.node, ss.ptr, ss.nnodes, ss.pid, ss.w, ss.series, F[0], m,
                    p->dev_ctr, ss.stride, ss.t0, pp);
    }
    case SDMP_ACT_INTERP: {
      const float* fld = resolve(p, I[2], I[3], time);
      const SparseSet& ss = p->sparse[I[4]];
      if (time < ss.t0) return SDMP_OK;
      return interpolate(st, fld, ss.node, ss.w, ss.npts, ss.ncorner, ss.series, p->dev_ctr,
                         ss.stride, ss.t0);
    }
    case SDMP_ACT_POST: {
      // [k,s, phase, nmsg, engine, msgs(12 each: fsrc,t,fdst,slo3,dlo3,ext3)..., nsig, (flags_id, slot)...]
      // I[4]: bit 0 engine (0 copy engine, 1 SM stores); bit 4: halos were
      // already pushed by the fused compute kernels, copy only on the first
      // step of a run (nothing was pushed before it)
      const int64_t phase = I[2];
      const int engine = (int)(I[4] & 3);  // 0 copy engines, 1 SM per box, 2 SM batched
      const bool pushed = (I[4] & 16) && time != p->run_time_m;
      const int64_t nmsg = pushed ? 0 : I[3];
      const int64_t* m = I + 5;
      const int fan = (engine == 0 && nmsg > 1) ? (int)(nmsg < sdmp_plan::kCopy ? nmsg
                                                                              : sdmp_plan::kCopy)
                                                : 1;
      if (fan > 1) {
        SDMP_CUDA(cudaEventRecord(p->ev_fork, st));
        for (int c = 0; c < fan; ++c) SDMP_CUDA(cudaStreamWaitEvent(p->cs[c], p->ev_fork, 0));
      }
      if (engine == 2) {
        // one kernel moves every box of the post (k_multi_copy)
        MultiCopy mc;
        for (int64_t q = 0; q < nmsg; ++q, m += 12) {
          SDMP_CHECK(mc.n < kMaxCopyMsgs, "too many messages for a batched post");
          const int64_t* sf = p->fields[m[0]].full;
          const int64_t* df = p->fields[m[2]].full;
          CopyMsg& c = mc.m[mc.n];
          c.src = resolve(p, m[0], m[1], time);
          c.dst = resolve(p, m[2], m[1], time);
          c.ssy = sf[2]; c.ssx = sf[1] * sf[2];
          c.dsy = df[2]; c.dsx = df[1] * df[2];
          c.soff = m[3] * c.ssx + m[4] * c.ssy + m[5];
          c.doff = m[6] * c.dsx + m[7] * c.dsy + m[8];
          c.ex = (int)m[9]; c.ey = (int)m[10]; c.ez = (int)m[11];
          if (c.ex <= 0 || c.ey <= 0 || c.ez <= 0) continue;
          mc.row0[mc.n] = mc.rows;
          mc.rows += (int64_t)c.ex * c.ey;
          ++mc.n;
        }
        int rc = multi_copy(st, mc);
        if (rc) return rc;
      }
      for (int64_t q = 0; engine != 2 && q < nmsg; ++q, m += 12) {
        const float* src = resolve(p, m[0], m[1], time);
        float* dst = resolve(p, m[2], m[1], time);
        cudaStream_t cst = fan > 1 ? p->cs[q % fan] : st;
        int rc = copy_box(cst, src, p->fields[m[0]].full, m + 3, dst, p->fields[m[2]].full,
                          m + 6, m + 9, engine);
        if (rc) return rc;
      }
      if (fan > 1) {
        for (int c = 0; c < fan; ++c) {
          SDMP_CUDA(cudaEventRecord(p->ev_cdone[c], p->cs[c]));
          SDMP_CUDA(cudaStreamWaitEvent(st, p->ev_cdone[c], 0));
        }
      }
      if (pushed) m = I + 5 + 12 * I[3];
      const int64_t nsig = *m++;
      uint32_t* ptrs[32];
      SDMP_CHECK(nsig <= 32, "too many signals");
      for (int64_t q = 0; q < nsig; ++q) ptrs[q] = p->flags[m[2 * q]] + m[2 * q + 1];
      return signal_flags(st, ptrs, (int)nsig, 0, p->dev_ctr, p->phases, (int)phase);
    }
    case SDMP_ACT_WAIT: {
      // [k,s, phase, nslot, slots...]
      const int64_t phase = I[2], n = I[3];
      SDMP_CHECK(p->local_flags != nullptr, "wait without local flags");
      SDMP_CHECK(n <= 32, "too many waits");
      uint32_t* ptrs[32];
      for (int64_t q = 0; q < n; ++q) ptrs[q] = p->local_flags + I[4 + q];
      return wait_flags(st, ptrs, (int)n, 0, (unsigned long long)p->timeout_ms * 1000000ull,
                        p->err_dev, p->dev_ctr, p->phases, (int)phase);
    }
    case SDMP_ACT_RECORD:
      SDMP_CHECK(I[2] >= 0 && I[2] < 32, "event id");
      SDMP_CUDA(cudaEventRecord(p->ev_user[I[2]], st));
      return SDMP_OK;
    case SDMP_ACT_STREAMWAIT:
      SDMP_CHECK(I[2] >= 0 && I[2] < 32, "event id");
      SDMP_CUDA(cudaStreamWaitEvent(st, p->ev_user[I[2]], 0));
      return SDMP_OK;
  }
  set_error("unknown plan action kind " + std::to_string(kind));
  return SDMP_EINVAL;
}

}  // namespace

// ---------------------------------------------------------------------------
// library

extern "C" const char* sdmp_last_error(void) { return get_error(); }
extern "C" int sdmp_version(void) { return 1; }

extern "C" int sdmp_device_count(int* n) {
  SDMP_CHECK(n, "null");
  cudaError_t e = cudaGetDeviceCount(n);
  if (e != cudaSuccess) {
    *n = 0;
    cudaGetLastError();
  }
  return SDMP_OK;
}

extern "C" int sdmp_device_info(int device, int* sm_count, int64_t* l2_bytes, int* cc_major,
                                int* cc_minor) {
  int v = 0;
  SDMP_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
  if (sm_count) *sm_count = v;
  SDMP_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, device));
  if (l2_bytes) *l2_bytes = v;
  SDMP_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMajor, device));
  if (cc_major) *cc_major = v;
  SDMP_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMinor, device));
  if (cc_minor) *cc_minor = v;
  return SDMP_OK;
}

// ---------------------------------------------------------------------------
// IPC

typedef CUresult (*PFN_getAddressRange)(CUdeviceptr*, size_t*, CUdeviceptr);

extern "C" int sdmp_ipc_export(const void* ptr, unsigned char handle[64], uint64_t* offset) {
  SDMP_CHECK(ptr && handle && offset, "null argument");
  static PFN_getAddressRange fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    SDMP_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", (void**)&fn, cudaEnableDefault, &q));
    SDMP_CHECK(fn && q == cudaDriverEntryPointSuccess, "cuMemGetAddressRange unavailable");
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  CUresult r = fn(&base, &size, (CUdeviceptr)ptr);
  if (r != CUDA_SUCCESS) {
    set_error("cuMemGetAddressRange failed: " + std::to_string((int)r));
    return SDMP_ECUDA;
  }
  cudaIpcMemHandle_t h;
  SDMP_CUDA(cudaIpcGetMemHandle(&h, (void*)base));
  static_assert(sizeof(h) == 64, "ipc handle size");
  std::memcpy(handle, &h, 64);
  *offset = (uint64_t)((CUdeviceptr)ptr - base);
  return SDMP_OK;
}

extern "C" int sdmp_ipc_import(const unsigned char handle[64], uint64_t offset, void** ptr) {
  SDMP_CHECK(handle && ptr, "null argument");
  static std::mutex mu;
  static std::map<std::string, void*> opened;
  std::lock_guard<std::mutex> lk(mu);
  std::string key((const char*)handle, 64);
  auto it = opened.find(key);
  void* base = nullptr;
  if (it != opened.end()) {
    base = it->second;
  } else {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    SDMP_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    opened[key] = base;
  }
  *ptr = (char*)base + offset;
  return SDMP_OK;
}

extern "C" int sdmp_flags_alloc(int32_t n, uint32_t** dptr) {
  SDMP_CHECK(n > 0 && dptr, "bad flags request");
  SDMP_CUDA(cudaMalloc((void**)dptr, n * sizeof(uint32_t)));
  SDMP_CUDA(cudaMemset(*dptr, 0, n * sizeof(uint32_t)));
  SDMP_CUDA(cudaDeviceSynchronize());
  return SDMP_OK;
}

extern "C" int sdmp_flags_free(uint32_t* dptr) {
  if (dptr) SDMP_CUDA(cudaFree(dptr));
  return SDMP_OK;
}

extern "C" int sdmp_enable_peer(int peer_device) {
  int can = 0, dev = 0;
  SDMP_CUDA(cudaGetDevice(&dev));
  if (peer_device == dev) return SDMP_OK;
  SDMP_CUDA(cudaDeviceCanAccessPeer(&can, dev, peer_device));
  SDMP_CHECK(can, "peer access not possible");
  cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return SDMP_OK;
  }
  SDMP_CUDA(e);
  return SDMP_OK;
}

// ---------------------------------------------------------------------------
// plan

extern "C" int sdmp_plan_create(int32_t device, int32_t phases_per_step, sdmp_plan** out) {
  SDMP_CHECK(out && phases_per_step >= 1, "bad plan arguments");
  SDMP_CUDA(cudaSetDevice(device));
  sdmp_plan* p = new sdmp_plan();
  p->device = device;
  p->phases = phases_per_step;
  int lo = 0, hi = 0;
  SDMP_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  SDMP_CUDA(cudaStreamCreateWithPriority(&p->s[0], cudaStreamNonBlocking, lo));
  SDMP_CUDA(cudaStreamCreateWithPriority(&p->s[1], cudaStreamNonBlocking, hi));
  SDMP_CUDA(cudaStreamCreateWithPriority(&p->s[2], cudaStreamNonBlocking, hi));
  SDMP_CUDA(cudaEventCreateWithFlags(&p->ev_step, cudaEventDisableTiming));
  for (int k = 0; k < 3; ++k) SDMP_CUDA(cudaEventCreateWithFlags(&p->ev_join[k], cudaEventDisableTiming));
  for (int k = 0; k < 32; ++k) SDMP_CUDA(cudaEventCreateWithFlags(&p->ev_user[k], cudaEventDisableTiming));
  SDMP_CUDA(cudaEventCreateWithFlags(&p->ev_in, cudaEventDisableTiming));
  SDMP_CUDA(cudaEventCreateWithFlags(&p->ev_out, cudaEventDisableTiming));
  SDMP_CUDA(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming));
  for (int c = 0; c < sdmp_plan::kCopy; ++c) {
    SDMP_CUDA(cudaStreamCreateWithPriority(&p->cs[c], cudaStreamNonBlocking, hi));
    SDMP_CUDA(cudaEventCreateWithFlags(&p->ev_cdone[c], cudaEventDisableTiming));
  }
  SDMP_CUDA(cudaMalloc((void**)&p->dev_ctr, 2 * sizeof(int64_t)));
  SDMP_CUDA(cudaMemset(p->dev_ctr, 0, 2 * sizeof(int64_t)));
  SDMP_CUDA(cudaHostAlloc((void**)&p->err_host, sizeof(int), cudaHostAllocMapped));
  *p->err_host = 0;
  SDMP_CUDA(cudaHostGetDevicePointer((void**)&p->err_dev, p->err_host, 0));
  *out = p;
  return SDMP_OK;
}

extern "C" int sdmp_plan_destroy(sdmp_plan* p) {
  if (!p) return SDMP_OK;
  cudaSetDevice(p->device);
  for (int k = 0; k < 3; ++k) {
    if (p->s[k]) cudaStreamSynchronize(p->s[k]);
  }
  for (int k = 0; k < 3; ++k) {
    if (p->s[k]) cudaStreamDestroy(p->s[k]);
    if (p->ev_join[k]) cudaEventDestroy(p->ev_join[k]);
  }
  for (int k = 0; k < 32; ++k) cudaEventDestroy(p->ev_user[k]);
  cudaEventDestroy(p->ev_step);
  cudaEventDestroy(p->ev_in);
  cudaEventDestroy(p->ev_out);
  cudaEventDestroy(p->ev_fork);
  for (int c = 0; c < sdmp_plan::kCopy; ++c) {
    if (p->cs[c]) {
      cudaStreamSynchronize(p->cs[c]);
      cudaStreamDestroy(p->cs[c]);
    }
    cudaEventDestroy(p->ev_cdone[c]);
  }
  for (auto e : p->tr_beg) cudaEventDestroy(e);
  for (auto e : p->tr_end) cudaEventDestroy(e);
  if (p->tr_origin) cudaEventDestroy(p->tr_origin);
  if (p->err_host) cudaFreeHost(p->err_host);
  for (auto& kv : p->graphs) cudaGraphExecDestroy(kv.second);
  if (p->dev_ctr) cudaFree(p->dev_ctr);
  delete p;
  return SDMP_OK;
}

extern "C" int sdmp_plan_add_field(sdmp_plan* p, int32_t nbuf, const uint64_t* ptrs,
                                   const int64_t full[3], int32_t* field_id) {
  SDMP_CHECK(p && ptrs && full && field_id, "null argument");
  SDMP_CHECK(nbuf >= 1 && nbuf <= 8, "nbuf must be 1..8");
  Field f;
  f.nbuf = nbuf;
  for (int k = 0; k < nbuf; ++k) {
    SDMP_CHECK(ptrs[k] != 0, "null buffer pointer");
    f.ptr[k] = ptrs[k];
  }
  for (int a = 0; a < 3; ++a) f.full[a] = full[a];
  p->fields.push_back(f);
  *field_id = (int32_t)p->fields.size() - 1;
  return SDMP_OK;
}

extern "C" int sdmp_plan_add_flags(sdmp_plan* p, uint32_t* flags, int32_t* flags_id) {
  SDMP_CHECK(p && flags && flags_id, "null argument");
  p->flags.push_back(flags);
  *flags_id = (int32_t)p->flags.size() - 1;
  return SDMP_OK;
}

extern "C" int sdmp_plan_set_local_flags(sdmp_plan* p, uint32_t* flags) {
  SDMP_CHECK(p && flags, "null argument");
  p->local_flags = flags;
  return SDMP_OK;
}

extern "C" int sdmp_plan_add_sparse(sdmp_plan* p, int32_t kind, int32_t npts, int32_t nnodes,
                                    int32_t ncorner, const int64_t* node_or_idx,
                                    const int32_t* ptr, const int32_t* pid, const float* w,
                                    float* series, int64_t series_stride, int64_t time_origin,
                                    int32_t* set_id) {
  SDMP_CHECK(p && set_id, "null argument");
  SDMP_CHECK(kind == 0 || kind == 1, "sparse kind must be 0 (inject) or 1 (interpolate)");
  SparseSet s{};
  s.kind = kind; s.npts = npts; s.nnodes = nnodes; s.ncorner = ncorner;
  s.node = node_or_idx; s.ptr = ptr; s.pid = pid; s.w = w; s.series = series;
  s.stride = series_stride; s.t0 = time_origin;
  p->sparse.push_back(s);
  *set_id = (int32_t)p->sparse.size() - 1;
  return SDMP_OK;
}

static int validate(const sdmp_plan* p, const Action& a) {
  const int64_t* I = a.i.data();
  const int n = (int)a.i.size();
  SDMP_CHECK(n >= 2, "action too short");
  SDMP_CHECK(I[1] >= 0 && I[1] < 3, "stream id must be 0..2");
  auto fchk = [&](int64_t f) { return f >= -1 && f < (int64_t)p->fields.size(); };
  static const std::map<int, int> min_len = {
      {SDMP_ACT_STAR, 19}, {SDMP_ACT_VSTAR, 21}, {SDMP_ACT_ROT, 23}, {SDMP_ACT_TTI, 33}, {SDMP_ACT_EL_V, 35}, {SDMP_ACT_EL_T, 43},
      {SDMP_ACT_VISCO_T, 69}, {SDMP_ACT_INJECT, 6}, {SDMP_ACT_INTERP, 5}, {SDMP_ACT_POST, 6},
      {SDMP_ACT_WAIT, 4}, {SDMP_ACT_RECORD, 3}, {SDMP_ACT_STREAMWAIT, 3}};
  auto it = min_len.find((int)I[0]);
  SDMP_CHECK(it != min_len.end(), "unknown action kind");
  SDMP_CHECK(n >= it->second, "action too short for its kind");
  switch ((int)I[0]) {
    case SDMP_ACT_STAR:
      SDMP_CHECK(fchk(I[2]) && I[2] >= 0 && fchk(I[4]) && fchk(I[6]) && fchk(I[7]) && I[7] >= 0,
                 "star: field id");
      SDMP_CHECK((int)a.f.size() >= 3 * SDMP_NCOEF + 3, "star: float params");
      break;
    case SDMP_ACT_VSTAR:
      SDMP_CHECK(fchk(I[2]) && I[2] >= 0 && fchk(I[4]) && fchk(I[6]) && I[6] >= 0 &&
                     fchk(I[7]) && fchk(I[8]) && I[8] >= 0 && fchk(I[9]) && I[9] >= 0,
                 "vstar: field id");
      SDMP_CHECK((int)a.f.size() >= 3 * SDMP_NCOEF, "vstar: float params");
      break;
    case SDMP_ACT_ROT:
      for (int k = 0; k < 7; ++k) SDMP_CHECK(fchk(I[2 + 2 * k]) && I[2 + 2 * k] >= 0, "rot: field id");
      SDMP_CHECK((int)a.f.size() >= 3 * SDMP_NCOEF + 1, "rot: float params");
      break;
    case SDMP_ACT_INJECT:
      SDMP_CHECK(I[5] >= 0 && I[5] < (int64_t)p->sparse.size(), "inject: set id");
      SDMP_CHECK(a.f.size() >= 1, "inject: float params");
      break;
    case SDMP_ACT_INTERP:
      SDMP_CHECK(I[4] >= 0 && I[4] < (int64_t)p->sparse.size(), "interp: set id");
      break;
    case SDMP_ACT_POST: {
      const int64_t nmsg = I[3];
      SDMP_CHECK(n >= 6 + 12 * nmsg, "post: truncated messages");
      const int64_t* m = I + 5;
      for (int64_t q = 0; q < nmsg; ++q, m += 12)
        SDMP_CHECK(fchk(m[0]) && m[0] >= 0 && fchk(m[2]) && m[2] >= 0, "post: field id");
      const int64_t nsig = *m++;
      SDMP_CHECK(n >= 6 + 12 * nmsg + 2 * nsig, "post: truncated signals");
      for (int64_t q = 0; q < nsig; ++q)
        SDMP_CHECK(m[2 * q] >= 0 && m[2 * q] < (int64_t)p->flags.size() && m[2 * q + 1] >= 0 &&
                       m[2 * q + 1] < 32, "post: flags id / slot");
      break;
    }
    case SDMP_ACT_WAIT:
      SDMP_CHECK(n >= 4 + I[3], "wait: truncated");
      for (int64_t q = 0; q < I[3]; ++q) SDMP_CHECK(I[4 + q] >= 0 && I[4 + q] < 32, "wait slot");
      break;
    default:
      break;
  }
  return SDMP_OK;
}

extern "C" int sdmp_plan_add_action(sdmp_plan* p, const int64_t* ints, int32_t nints,
                                    const float* floats, int32_t nfloats) {
  SDMP_CHECK(p && ints && nints > 0, "null argument");
  Action a;
  a.i.assign(ints, ints + nints);
  if (floats && nfloats > 0) a.f.assign(floats, floats + nfloats);
  int rc = validate(p, a);
  if (rc) return rc;
  p->actions.push_back(std::move(a));
  return SDMP_OK;
}

extern "C" int sdmp_plan_set_timeout(sdmp_plan* p, int64_t ms) {
  SDMP_CHECK(p && ms > 0, "bad timeout");
  p->timeout_ms = ms;
  return SDMP_OK;
}

extern "C" int sdmp_plan_set_tracing(sdmp_plan* p, int32_t on) {
  SDMP_CHECK(p, "null plan");
  p->tracing = on != 0;
  return SDMP_OK;
}

// events for (step s, action k): begin at 2*(s*nact+k), end at +1; one
// origin event per step (recorded on stream 0 at the step start)
static int trace_events(sdmp_plan* p, int64_t steps) {
  const size_t need = (size_t)(2 * steps * p->actions.size());
  while (p->tr_beg.size() < need) {
    cudaEvent_t e;
    SDMP_CUDA(cudaEventCreate(&e));
    p->tr_beg.push_back(e);
  }
  while (p->tr_end.size() < (size_t)steps) {
    cudaEvent_t e;
    SDMP_CUDA(cudaEventCreate(&e));
    p->tr_end.push_back(e);
  }
  return SDMP_OK;
}

extern "C" int sdmp_plan_set_graph(sdmp_plan* p, int32_t on) {
  SDMP_CHECK(p, "null plan");
  p->graph_on = on != 0;
  // replay period = lcm of the buffer counts (rotation repeats after it)
  int per = 1;
  for (const auto& f : p->fields) {
    int a = per, b = f.nbuf;
    while (b) { int t = a % b; a = b; b = t; }
    per = per / a * f.nbuf;
  }
  p->period = per;
  return SDMP_OK;
}

// Enqueue one timestep.  `si` >= 0 records tracing events for step slot si.
static int enqueue_step(sdmp_plan* p, int64_t time, int64_t si) {
  const size_t nact = p->actions.size();
  SDMP_CUDA(cudaEventRecord(p->ev_step, p->s[0]));
  SDMP_CUDA(cudaStreamWaitEvent(p->s[1], p->ev_step, 0));
  SDMP_CUDA(cudaStreamWaitEvent(p->s[2], p->ev_step, 0));
  if (si >= 0) SDMP_CUDA(cudaEventRecord(p->tr_end[si], p->s[0]));
  for (size_t k = 0; k < nact; ++k) {
    cudaStream_t st = p->s[p->actions[k].i[1]];
    if (si >= 0) SDMP_CUDA(cudaEventRecord(p->tr_beg[2 * (si * nact + k)], st));
    int rc = run_action(p, p->actions[k], time);
    if (rc) return rc;
    if (si >= 0) SDMP_CUDA(cudaEventRecord(p->tr_beg[2 * (si * nact + k) + 1], st));
  }
  SDMP_CUDA(cudaEventRecord(p->ev_join[1], p->s[1]));
  SDMP_CUDA(cudaEventRecord(p->ev_join[2], p->s[2]));
  SDMP_CUDA(cudaStreamWaitEvent(p->s[0], p->ev_join[1], 0));
  SDMP_CUDA(cudaStreamWaitEvent(p->s[0], p->ev_join[2], 0));
  return tick_ctr(p->s[0], p->dev_ctr);
}

// Capture `period` steps starting at a time with residue r into a graph.
static int capture_period(sdmp_plan* p, int64_t time, cudaGraphExec_t* out) {
  cudaGraph_t g = nullptr;
  SDMP_CUDA(cudaStreamBeginCapture(p->s[0], cudaStreamCaptureModeRelaxed));
  int rc = SDMP_OK;
  for (int k = 0; k < p->period && rc == SDMP_OK; ++k) rc = enqueue_step(p, time + k, -1);
  cudaError_t e = cudaStreamEndCapture(p->s[0], &g);
  if (rc) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  SDMP_CUDA(e);
  cudaError_t ei = cudaGraphInstantiate(out, g, 0);
  cudaGraphDestroy(g);
  SDMP_CUDA(ei);
  return SDMP_OK;
}

extern "C" int sdmp_plan_run(sdmp_plan* p, int64_t time_m, int64_t time_M, void* stream) {
  SDMP_CHECK(p, "null plan");
  SDMP_CHECK(time_M >= time_m - 1, "time_M < time_m - 1");
  SDMP_CUDA(cudaSetDevice(p->device));
  cudaStream_t user = (cudaStream_t)stream;
  const int64_t nsteps = time_M - time_m + 1;
  if (p->tracing && nsteps > 0) {
    int rc = trace_events(p, nsteps);
    if (rc) return rc;
  }
  SDMP_CUDA(cudaEventRecord(p->ev_in, user));
  SDMP_CUDA(cudaStreamWaitEvent(p->s[0], p->ev_in, 0));
  int rc = set_ctr(p->s[0], p->dev_ctr, time_m, p->steps_done);
  if (rc) return rc;
  p->run_time_m = time_m;
  int64_t time = time_m;
  // graphs: only after the plan has run once (lazy attributes, scratch
  // allocations and TMA descriptor entry points are resolved by then)
  const bool graphs = p->graph_on && !p->tracing && p->period >= 1 && p->steps_done > 0;
  while (time <= time_M) {
    const int64_t left = time_M - time + 1;
    if (graphs && time > time_m && left >= p->period) {
      const int64_t r = ((time % p->period) + p->period) % p->period;
      auto it = p->graphs.find(r);
      if (it == p->graphs.end()) {
        cudaGraphExec_t ex = nullptr;
        rc = capture_period(p, time, &ex);
        if (rc) return rc;
        it = p->graphs.emplace(r, ex).first;
      }
      SDMP_CUDA(cudaGraphLaunch(it->second, p->s[0]));
      time += p->period;
      p->steps_done += p->period;
      continue;
    }
    rc = enqueue_step(p, time, p->tracing ? time - time_m : -1);
    if (rc) return rc;
    time += 1;
    p->steps_done += 1;
  }
  p->last_traced = p->tracing ? (int)nsteps : 0;
  SDMP_CUDA(cudaEventRecord(p->ev_out, p->s[0]));
  SDMP_CUDA(cudaStreamWaitEvent(user, p->ev_out, 0));
  return SDMP_OK;
}

extern "C" int sdmp_plan_step(sdmp_plan* p, int64_t time, void* stream) {
  return sdmp_plan_run(p, time, time, stream);
}

extern "C" int sdmp_plan_sync(sdmp_plan* p) {
  SDMP_CHECK(p, "null plan");
  SDMP_CUDA(cudaSetDevice(p->device));
  for (int k = 0; k < 3; ++k) SDMP_CUDA(cudaStreamSynchronize(p->s[k]));
  if (*p->err_host) {
    *p->err_host = 0;
    set_error("halo wait exceeded the watchdog (" + std::to_string(p->timeout_ms) +
              " ms): a neighbour rank did not deliver its halo");
    return SDMP_ETIMEOUT;
  }
  return SDMP_OK;
}

// rows (6 per action): {index, stream, kind, mean start ms (from the step
// start on stream 0), mean duration ms, launches per step}, averaged over
// every step of the last traced run.
extern "C" int sdmp_plan_trace(sdmp_plan* p, double* rows, int32_t max_rows, int32_t* nrows) {
  SDMP_CHECK(p && rows && nrows, "null argument");
  SDMP_CUDA(cudaSetDevice(p->device));
  const int64_t nsteps = p->last_traced;
  const size_t nact = p->actions.size();
  int n = 0;
  for (size_t k = 0; k < nact && n < max_rows && nsteps > 0; ++k, ++n) {
    double sb = 0.0, sd = 0.0;
    for (int64_t s = 0; s < nsteps; ++s) {
      float b = 0.f, e = 0.f;
      SDMP_CUDA(cudaEventElapsedTime(&b, p->tr_end[s], p->tr_beg[2 * (s * nact + k)]));
      SDMP_CUDA(cudaEventElapsedTime(&e, p->tr_end[s], p->tr_beg[2 * (s * nact + k) + 1]));
      sb += b;
      sd += e - b;
    }
    rows[6 * n + 0] = (double)k;
    rows[6 * n + 1] = (double)p->actions[k].i[1];
    rows[6 * n + 2] = (double)p->actions[k].i[0];
    rows[6 * n + 3] = sb / nsteps;
    rows[6 * n + 4] = sd / nsteps;
    rows[6 * n + 5] = (double)launches_of(p->actions[k]);
  }
  *nrows = n;
  return SDMP_OK;
}
