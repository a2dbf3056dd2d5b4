/*
 * sdmp.h — C ABI of the B200 finite-difference propagator path
 * (libsdmp.so, built from paper_2312_13094_b200/csrc for sm_100a).
 *
 * The reference (arXiv 2312.13094 artifact, /root/reference) is Python and
 * specifies its runtime only as prose contracts in SPEC.md; every entry
 * point below names the SPEC operation it replaces.  The Python host layer
 * (paper_2312_13094_b200/runtime.py) binds these with ctypes; INTEGRATION.md
 * shows the binding a maintainer of the reference would add.
 *
 * Conventions
 *  - All functions return 0 (SDMP_OK) or a negative status; the message of
 *    the last failure on the calling thread is sdmp_last_error().
 *  - Arrays are fp32, row-major, FULL layout (DOMAIN + halo per side,
 *    SPEC.md:214-217): element (x, y, z) at x*full[1]*full[2] + y*full[2] + z.
 *  - Boxes are half-open [lo, hi) in FULL coordinates (after
 *    align_accesses).
 *  - `stream` is a cudaStream_t passed as void* (0 = legacy default stream).
 *    Kernel entry points are asynchronous and stream-ordered.
 *  - No torch / C++ types cross this boundary.
 */
#ifndef SDMP_H
#define SDMP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    SDMP_OK = 0,
    SDMP_EINVAL = -1,      /* bad argument (message names it) */
    SDMP_ECUDA = -2,       /* CUDA runtime / driver error */
    SDMP_ETIMEOUT = -3,    /* halo wait exceeded the watchdog */
    SDMP_EUNSUPPORTED = -4 /* configuration not compiled in */
};

#define SDMP_MAX_RADIUS 8   /* SO 16 */
#define SDMP_NCOEF (SDMP_MAX_RADIUS + 1)

/* ---- library --------------------------------------------------------- */
const char* sdmp_last_error(void);
int sdmp_version(void);
int sdmp_device_count(int* n);
/* Device properties needed by the host planner: SM count, L2 bytes. */
int sdmp_device_info(int device, int* sm_count, int64_t* l2_bytes, int* cc_major, int* cc_minor);

/* ---- stencil kernels: compute(box, equation) ---- */

/* Star stencil family, replaces compute() for the acoustic kernel
 * (solved form symbolics.py:629-674) and the diffusion
 * kernel:
 *     u1 = A*u0 + B*u2 + S * L(u0),   S = C / m  (m != NULL) or C,
 *     L(u0) = sum_a [c_a0 u0 + sum_k c_ak (u0[-k e_a] + u0[+k e_a])].
 * coeffs: 3 * SDMP_NCOEF floats, axis-major, c_ak = w_k / h_a^2 bound to
 * fp32 once.  radius[a] in 0..8.  u2 may be NULL when B == 0.
 * variant (low byte): 0 auto, 1 generic (one thread per point),
 * 2 streaming (register x-window + shared-memory y/z plane), 3 TMA pipeline
 * (cp.async.bulk.tensor ring + mbarriers; the auto choice).  2 and 3 need
 * equal radii and 4-aligned z (FULL z, box z); otherwise generic runs.
 * Flag SDMP_VARIANT_M_IS_SCALE: `m` already holds S = C/m (see
 * sdmp_bind_scale), so the kernel multiplies instead of dividing. */
#define SDMP_VARIANT_M_IS_SCALE 0x100
int sdmp_star_update(void* stream, const float* u0, const float* u2, const float* m,
                     float* u1, const int64_t full[3], const int64_t lo[3],
                     const int64_t hi[3], const int32_t radius[3], const float* coeffs,
                     float A, float B, float C, int32_t variant);

/* Variable-coefficient star (acoustic with an absorbing / damping layer and
 * other updates whose coefficients depend on static fields):
 *   u1 = A u0 + B u2 + S L(u0)
 * with per-point A, B, S arrays (FULL-shaped like u, read at the output
 * point; B may be NULL, then u2 is unused).  Replaces compute(box, eq) for
 * the reference's solved `m*u.dt2 - u.laplace + damp*u.dt` (symbolics.py
 * solve_forward); coefficients are bound once per apply by the
 * host from the solved update.  variant 1 forces the generic kernel. */
int sdmp_var_star_update(void* stream, const float* u0, const float* u2, const float* A,
                         const float* B, const float* S, float* u1, const int64_t full[3],
                         const int64_t lo[3], const int64_t hi[3], const int32_t radius[3],
                         const float* coeffs, int32_t variant);

/* Bind a derived fp32 parameter once at plan build:
 * out[i] = in[i] != 0 ? C / in[i] : 0 for n elements (e.g. S = dt^2/m). */
int sdmp_bind_scale(void* stream, float* out, const float* in, int64_t n, float C);

/* Pseudo-acoustic TTI (SPEC.md:594-601 nested D^T D):
 * in[] = {p0, p2, r0, r2, m, epsp, delp, ax, ay, az}; out p1, r1.
 * lap_c, d1_c: 3 * SDMP_NCOEF (d1_c[a*NCOEF + k] = w1_k / h_a, k >= 1).
 * Reads p0/r0 up to 2*radius (= SO) from each point, ax/ay/az up to radius.
 * radius | SDMP_VARIANT_M_IS_SCALE: the m operand holds the bound scale
 * dt2/m (sdmp_bind_scale) instead of m (same results). */
int sdmp_tti_update(void* stream, const float* const in[10], float* p1, float* r1,
                    const int64_t full[3], const int64_t lo[3], const int64_t hi[3],
                    int32_t radius, const float* lap_c, const float* d1_c, float dt2,
                    int32_t variant);

/* Single-field rotated operator (the SPEC's tti_gxx_kernel):
 * m u_tt = G u with G u = sum_i D_i(a_i sum_j a_j D_j u) (nested centred first
 * derivatives), solved u1 = 2 u0 - u2 + dt2/m G u0.  in[] = {u0, u2, m, ax,
 * ay, az}; d1_c as for sdmp_tti_update; reads u0 up to 2*radius;
 * radius | SDMP_VARIANT_M_IS_SCALE as for sdmp_tti_update. */
int sdmp_rot_update(void* stream, const float* const in[6], float* u1, const int64_t full[3],
                    const int64_t lo[3], const int64_t hi[3], int32_t radius,
                    const float* d1_c, float dt2);

/* Staggered velocity-stress elastic / viscoelastic.
 * sc: 3 * SDMP_MAX_RADIUS staggered weights / h_a (k = 1..radius).
 * v = {vx, vy, vz}; tau = {xx, yy, zz, xy, xz, yz}. */
int sdmp_elastic_velocity(void* stream, const float* const v0[3], const float* const tau[6],
                          const float* b, float* const v1[3], const int64_t full[3],
                          const int64_t lo[3], const int64_t hi[3], int32_t radius,
                          const float* sc, float dt);
int sdmp_elastic_stress(void* stream, const float* const v1[3], const float* const t0[6],
                        const float* lam, const float* mu, float* const t1[6],
                        const int64_t full[3], const int64_t lo[3], const int64_t hi[3],
                        int32_t radius, const float* sc, float dt);
/* params = {l2m = pi*tau_ep/tau_s, mus = mu*tau_es/tau_s, its = 1/tau_s} */
/* The SPEC's collocated elastic_kernel: the same
 * velocity-stress system with centred first derivatives on one grid;
 * c1: 3 * SDMP_MAX_RADIUS central first-derivative weights / h_a (k = 1..R). */
int sdmp_elastic_colloc_velocity(void* stream, const float* const v0[3],
                                 const float* const tau[6], const float* b, float* const v1[3],
                                 const int64_t full[3], const int64_t lo[3], const int64_t hi[3],
                                 int32_t radius, const float* c1, float dt);
int sdmp_elastic_colloc_stress(void* stream, const float* const v1[3], const float* const t0[6],
                               const float* lam, const float* mu, float* const t1[6],
                               const int64_t full[3], const int64_t lo[3], const int64_t hi[3],
                               int32_t radius, const float* c1, float dt);
int sdmp_visco_stress(void* stream, const float* const v1[3], const float* const s0[6],
                      const float* const r0[6], const float* const params[3],
                      float* const s1[6], float* const r1[6], const int64_t full[3],
                      const int64_t lo[3], const int64_t hi[3], int32_t radius,
                      const float* sc, float dt);

/* ---- sparse ------------------------------------------ */

/* inject: for node i, acc = sum_{j in [ptr[i], ptr[i+1])} w[j] * amps[pid[j]]
 * (sequential in point-id order, no atomics), then
 * field[node[i]] += acc * (m ? C / m[node[i]] : C). */
int sdmp_inject(void* stream, float* field, const int64_t* node, const int32_t* ptr,
                int32_t nnodes, const int32_t* pid, const float* w, const float* amps,
                float C, const float* m);
/* interpolate: out[p] = sum_c w[p*ncorner+c] * field[idx[p*ncorner+c]]. */
int sdmp_interpolate(void* stream, const float* field, const int64_t* idx, const float* w,
                     int32_t npts, int32_t ncorner, float* out);

/* ---- halo data movement ------------------------------ */

/* pack_region / unpack_region: row-major box <-> contiguous buffer. */
int sdmp_pack(void* stream, const float* field, const int64_t full[3], const int64_t lo[3],
              const int64_t hi[3], float* buf);
int sdmp_unpack(void* stream, float* field, const int64_t full[3], const int64_t lo[3],
                const int64_t hi[3], const float* buf);
/* Box copy between two FULL arrays (either may be a peer/IPC pointer).
 * engine 0: copy engine (cudaMemcpy3DAsync); 1: SM kernel (peer stores);
 * 2: the batched post kernel of diagonal / basic mode, one box (16-byte
 * peer stores, one warp per z row). */
int sdmp_copy_box(void* stream, const float* src, const int64_t src_full[3],
                  const int64_t src_lo[3], float* dst, const int64_t dst_full[3],
                  const int64_t dst_lo[3], const int64_t extent[3], int32_t engine);

/* ---- inter-process memory (replaces the SPEC Transport) */
int sdmp_ipc_export(const void* ptr, unsigned char handle[64], uint64_t* offset);
int sdmp_ipc_import(const unsigned char handle[64], uint64_t offset, void** ptr);
int sdmp_flags_alloc(int32_t n, uint32_t** dptr);
int sdmp_flags_free(uint32_t* dptr);
int sdmp_enable_peer(int peer_device);

/* ---- plan executor (execute_plan_full / halo_exchange loop,
 *      SPEC.md:440-458; ExecPlan SPEC.md:310-315) ------------------------
 * A plan is an ordered per-timestep action list built by the host planner
 * (paper_2312_13094_b200/compiler.py) and replayed for time_m..time_M on
 * three streams (0 compute, 1 remainder [high priority], 2 exchange). */
typedef struct sdmp_plan sdmp_plan;

enum {
    SDMP_ACT_STAR = 1, SDMP_ACT_TTI = 2, SDMP_ACT_EL_V = 3, SDMP_ACT_EL_T = 4,
    SDMP_ACT_VISCO_T = 5, SDMP_ACT_INJECT = 6, SDMP_ACT_INTERP = 7, SDMP_ACT_VSTAR = 8, SDMP_ACT_ROT = 9,
    SDMP_ACT_POST = 10, SDMP_ACT_WAIT = 11, SDMP_ACT_RECORD = 12, SDMP_ACT_STREAMWAIT = 13,
    SDMP_ACT_PACK = 14, SDMP_ACT_UNPACK = 15
};

int sdmp_plan_create(int32_t device, int32_t phases_per_step, sdmp_plan** out);
int sdmp_plan_destroy(sdmp_plan* plan);
/* Register a (local or peer) field: nbuf device pointers, FULL shape. */
int sdmp_plan_add_field(sdmp_plan* plan, int32_t nbuf, const uint64_t* ptrs,
                        const int64_t full[3], int32_t* field_id);
/* Register the receive-flag array of a peer (IPC pointer) -> flags id. */
int sdmp_plan_add_flags(sdmp_plan* plan, uint32_t* flags, int32_t* flags_id);
/* Local flags (written by peers), waited on by SDMP_ACT_WAIT. */
int sdmp_plan_set_local_flags(sdmp_plan* plan, uint32_t* flags);
/* Sparse set: device arrays for inject (node/ptr/pid/w, amps[nt*npts]) or
 * interpolate (idx/w, out[nt*npts]); returns set id. */
int sdmp_plan_add_sparse(sdmp_plan* plan, int32_t kind, int32_t npts, int32_t nnodes,
                         int32_t ncorner, const int64_t* node_or_idx, const int32_t* ptr,
                         const int32_t* pid, const float* w, float* series,
                         int64_t series_stride, int64_t time_origin, int32_t* set_id);
/* Append one action: ints = {kind, stream, ...} (see compiler.py for the
 * per-kind layout), floats = kind parameters. */
int sdmp_plan_add_action(sdmp_plan* plan, const int64_t* ints, int32_t nints,
                         const float* floats, int32_t nfloats);
/* Run time_m..time_M (inclusive) ordered after / before
 * `stream`.  Asynchronous. */
int sdmp_plan_run(sdmp_plan* plan, int64_t time_m, int64_t time_M, void* stream);
/* One timestep (= sdmp_plan_run(plan, time, time, stream)); the SURVEY's
 * proposed `sdmp_step` for per-step instrumentation. */
int sdmp_plan_step(sdmp_plan* plan, int64_t time, void* stream);
/* Block until the plan's streams drain; checks the halo watchdog. */
int sdmp_plan_sync(sdmp_plan* plan);
/* Per-action instrumentation: enable (records CUDA events around every
 * action of every step, on the action's stream) and read 6 doubles per
 * action {index, stream, kind, mean start ms from the step start, mean
 * duration ms, kernel launches per step} averaged over the last run. */
int sdmp_plan_set_tracing(sdmp_plan* plan, int32_t on);
int sdmp_plan_trace(sdmp_plan* plan, double* rows, int32_t max_rows, int32_t* nrows);
/* Watchdog for halo waits in milliseconds (default 30000). */
int sdmp_plan_set_timeout(sdmp_plan* plan, int64_t ms);
/* Capture one buffer-rotation period into a CUDA graph and replay it. */
int sdmp_plan_set_graph(sdmp_plan* plan, int32_t on);

#ifdef __cplusplus
}
#endif
#endif /* SDMP_H */
