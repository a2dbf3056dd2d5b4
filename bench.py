"""Benchmark: GPts/s of the FD propagator hot path on 1..8 B200s.

Workload (BASELINE.json configs[1]): 3D isotropic acoustic, SO-8, 1024^3
grid points PER GPU (weak scaling), global (1024 P, 1024 Q, 1024) on the
x/y topology (P, Q, 1) = (1,1,1) / (2,1,1) / (2,2,1) / (4,2,1), Ricker point
source at the global centre and a receiver line along x crossing ranks,
mpi mode ``full`` (override with --mode).  A "step" is one timestep over the
whole grid.  Synthetic velocity model (layered vp + hashed 1% noise).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--mode full]
    torchrun --nproc-per-node N bench.py --gpus N ...
    python bench.py --impl reference ...     # CPU oracle arm (rank 0 only)

Prints ONE JSON line (rank 0).  ``value`` = whole-job grid-point updates per
second (device-timed with CUDA events, max over ranks); ``e2e`` = the same
metric through ``Operator.apply`` with the source samples uploaded from host
memory and the receiver traces read back every step.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

TOPOS = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (4, 2, 1)}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="full")
    ap.add_argument("--so", type=int, default=8)
    ap.add_argument("--n", type=int, default=1024, help="grid points per axis per GPU")
    ap.add_argument("--nrec", type=int, default=256)
    ap.add_argument("--kernel", default="acoustic",
                    choices=["acoustic", "damped", "rotated", "tti", "elastic", "elastic_col",
                             "visco"])
    ap.add_argument("--shape", default=None, help="override the global shape nx,ny,nz")
    ap.add_argument("--topology", default=None,
                    help="override the rank grid px,py,pz (default 1,1,1 / 2,1,1 / 2,2,1 / 4,2,1)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    return ap.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = f"/tmp/sdmp_clocks_{os.getpid()}.csv"

    def start(self):
        """Start sampling and wait (<= 3 s) for the first sample, so the
        timed region that follows is covered (the sample taken just before
        it is kept as well: short regions still carry a reading)."""
        self.n0 = 0
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
            return
        t0 = time.time()
        while time.time() - t0 < 3.0:
            try:
                n = sum(1 for _ in open(self.path))
            except OSError:
                n = 0
            if n:
                self.n0 = n - 1
                return
            time.sleep(0.01)

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in list(open(self.path))[self.n0:]:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    mx = float(parts[2])
                except ValueError:
                    continue
                for nm, v in zip(names, parts[5:9]):
                    if v.lower() in ("active", "1"):
                        reasons.add(nm)
        except Exception:
            return None
        if not sm:
            return None
        load = [s for s in sm if mx and s > 0.5 * mx] or sm
        return {"sm_mhz": float(np.median(load)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


class NvlinkCounters:
    """NVLink data bytes sent / received by this rank's GPU over an interval
    (NVML field values, cumulative per link, summed over links): the
    driver-side measurement of the halo traffic, independent of the
    library's own byte count.  None when NVML does not expose them."""

    def __init__(self, device):
        self.ok = False
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(device)
            self.ok = True
        except Exception:
            self.ok = False

    def read(self):
        if not self.ok:
            return None
        N = self.N
        out = {}
        for name, fid in (("tx", N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX),
                          ("rx", N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX)):
            total, ok = 0, 0
            try:
                # scopeId = link id; links that do not exist return an error
                vals = N.nvmlDeviceGetFieldValues(self.h, [(fid, link) for link in range(18)])
                for v in vals:
                    if v.nvmlReturn == 0:
                        total += int(v.value.ullVal)
                        ok += 1
            except Exception:
                return None
            if ok == 0:
                return None  # NOT_SUPPORTED (e.g. counters hidden on this box)
            out[name] = total * 1024  # the THROUGHPUT_DATA fields count KiB
            out[name + "_links"] = ok
        return out


# ---------------------------------------------------------------------------
# CPU reference arm / baseline: the oracle port (numpy, fp64) on a slab


class CpuSlab:
    """The oracle port of one configured step (oracle/stencils: star update,
    source injection, receiver interpolation -- the CPU restatement of the
    reference path) on a bounded slab of the n^3 workload: x-planes [0, nx)
    of the full n x n cross-section with a Ricker source and a receiver line
    inside the slab.  Arrays are allocated and filled ONCE (``__init__``);
    ``step()`` is the timed unit.  Threads split the slab along x (numpy
    releases the GIL)."""

    def __init__(self, n, so, threads=None, nx=None, nrec=256):
        from concurrent.futures import ThreadPoolExecutor
        from oracle import stencils as K
        from paper_2312_13094_b200.symbolics import fd_coefficients
        self.K = K
        self.so, r = so, so // 2
        self.threads = threads or os.cpu_count() or 1
        w = [float(c) for c in fd_coefficients(2, so)]
        self.h = h = 10.0
        self.coeffs = [np.float32([w[r + k] / (h * h) for k in range(r + 1)]).astype(np.float64)] * 3
        self.nx = nx or max(self.threads * 2, 8)
        self.ny = self.nz = n
        full = (self.nx + 2 * so, n + 2 * so, n + 2 * so)
        rng = np.random.default_rng(0)
        self.bufs = [rng.standard_normal(full) for _ in range(3)]
        self.m = np.full(full, 0.25)
        self.dt2 = 1e-3
        self.chunks = [c for c in np.array_split(np.arange(so, so + self.nx), self.threads) if len(c)]
        self.pool = ThreadPoolExecutor(self.threads)
        shape = (self.nx, n, n)
        ext = [h * (s_ - 1) for s_ in shape]
        src = [0.5 * ext[0] + 0.3, 0.5 * ext[1] + 3.7, 0.5 * ext[2] + 3.7]
        corners, weights = K.trilinear(src, (h, h, h), shape)
        self.src_nodes = {c: [(0, wt)] for c, wt in zip(corners, weights)}
        self.rec = [K.trilinear([x, 0.5 * ext[1] + 2.5, 20.3], (h, h, h), shape)
                    for x in np.linspace(5.0, ext[0] - 5.0, nrec)]
        self.amps = np.float32(K.ricker(0.010, np.arange(4096) * 1.0, 100.0)).astype(np.float64)
        self.time = 0
        self.trace = np.zeros(nrec)

    def step(self):
        K, so = self.K, self.so
        u2, u0, u1 = (self.bufs[(self.time + k) % 3] for k in (-1, 0, 1))
        halo, origin = (so, so, so), (0, 0, 0)
        for i, (c, wts) in enumerate(self.rec):   # receivers sample u[t]
            self.trace[i] = K.interpolate(u0, halo, origin, c, wts)

        def work(ix):
            box = ((int(ix[0]), so, so), (int(ix[-1]) + 1, so + self.ny, so + self.nz))
            K.star_update(u0, u2, self.m, self.coeffs, 2.0, -1.0, self.dt2, box, u1)

        list(self.pool.map(work, self.chunks))
        K.inject(u1, halo, origin, self.src_nodes, [self.amps[self.time % len(self.amps)]],
                 (self.dt2, self.m))
        self.time += 1

    @property
    def points(self):
        return self.nx * self.ny * self.nz

    def sample(self, reps, el):
        return (f"acoustic SO-{self.so} step (star update + Ricker injection + "
                f"{len(self.rec)}-receiver interpolation) on a {self.nx}x{self.ny}x{self.nz} "
                f"slab of the {self.ny}^3 per-GPU grid, {reps} steps in {el:.1f} s, numpy fp64 "
                f"oracle (oracle/stencils), {self.threads} threads; arrays allocated once, "
                f"outside the timed loop")

    def close(self):
        self.pool.shutdown()


def cpu_reference(n, so, seconds):
    """cpu_baseline: CpuSlab steps for ~``seconds`` (after one untimed step)."""
    slab = CpuSlab(n, so)
    slab.step()
    t0 = time.perf_counter()
    reps = 0
    while True:
        slab.step()
        reps += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    slab.close()
    return {"value": slab.points * reps / el / 1e9, "unit": "GPts/s", "cores": slab.threads,
            "kind": "port", "sample": slab.sample(reps, el)}


def run_reference(args):
    """--impl reference: the oracle port (the reference's CPU path restated;
    the reference itself ships no runtime to install) on the host cores.
    Each step = one CpuSlab step, W untimed then K timed; rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    slab = CpuSlab(args.n, args.so)
    for _ in range(max(args.warmup, 0)):
        slab.step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        slab.step()
    el = time.perf_counter() - t0
    slab.close()
    val = slab.points * args.steps / el / 1e9
    line = {"metric": "GPts/s", "value": val, "unit": "GPts/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"acoustic SO-{args.so} {args.n}^3 per GPU (configs[1]); CPU "
                                   "oracle on a bounded slab per step",
                       "points_per_step": slab.points, "mode": args.mode},
            "cpu_baseline": {"value": val, "unit": "GPts/s", "cores": slab.threads,
                             "kind": "port", "sample": slab.sample(args.steps, el)},
            "e2e": {"value": val, "unit": "GPts/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.warmup < 1:
        raise SystemExit("--warmup must be >= 1 (the first run binds the plan's derived buffers)")
    from paper_2312_13094_b200.dist import default_backend
    if world > 1 and not dist.is_initialized():
        local = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
        torch.cuda.set_device(local)
        backend = default_backend()
        kw = {"device_id": torch.device("cuda", local)} if backend == "nccl" else {}
        dist.init_process_group(backend, **kw)
    from paper_2312_13094_b200 import Grid, Operator, SparseTimeFunction
    from paper_2312_13094_b200 import kernels as KD
    from paper_2312_13094_b200 import symbolics as S
    from paper_2312_13094_b200.dist import context

    ctx = context()
    N = ctx.size
    if N not in TOPOS:
        raise SystemExit(f"unsupported GPU count {N}")
    topo = TOPOS[N] if not args.topology else tuple(int(x) for x in args.topology.split(","))
    if math.prod(topo) != N:
        raise SystemExit(f"topology {topo} does not match {N} ranks")
    n = args.n
    shape = tuple(n * p for p in topo)
    if args.shape:
        shape = tuple(int(x) for x in args.shape.split(","))
    h = 10.0
    grid = Grid(shape, tuple(h * (s - 1) for s in shape), topology=topo)
    GW = 8  # extra untimed steps: capture the CUDA graphs of every buffer-rotation phase
    total_steps = args.warmup + GW + args.steps
    nt = total_steps + 1
    ext = grid.extent
    src = KD.point_source(grid, [tuple(0.5 * e + 3.7 for e in ext)], nt, 1.0, f0=0.010)
    rec = KD.receiver_line(grid, args.nrec, nt)
    kname = args.kernel
    if kname == "acoustic":
        kd = KD.acoustic_model(grid, so=args.so)
        u, m = kd.fields["u"], kd.fields["m"]
        dt = float(np.float32(KD.critical_dt(4.6, grid.spacing)))
        terms = [src.inject(u.forward, expr=src * S.DT ** 2 / m), rec.interpolate(u)]
    elif kname == "damped":
        kd = KD.damped_acoustic_model(grid, so=args.so, nbl=40)
        u, m = kd.fields["u"], kd.fields["m"]
        dt = float(np.float32(KD.critical_dt(4.6, grid.spacing)))
        terms = [src.inject(u.forward, expr=src * S.DT ** 2 / m), rec.interpolate(u)]
    elif kname == "rotated":
        kd = KD.rotated_model(grid, so=args.so)
        u, m = kd.fields["u"], kd.fields["m"]
        dt = float(np.float32(KD.critical_dt(4.6, grid.spacing, 0.25)))
        terms = [src.inject(u.forward, expr=src * S.DT ** 2 / m), rec.interpolate(u)]
    elif kname == "tti":
        kd = KD.tti_model(grid, so=args.so)
        p, r, m = kd.fields["p"], kd.fields["r"], kd.fields["m"]
        dt = float(np.float32(KD.critical_dt(4.6, grid.spacing, 0.25)))
        src2 = KD.point_source(grid, src.coordinates, nt, 1.0, f0=0.010, name="src_r")
        terms = [src.inject(p.forward, expr=src * S.DT ** 2 / m),
                 src2.inject(r.forward, expr=src2 * S.DT ** 2 / m), rec.interpolate(p)]
    else:
        kd = (KD.viscoelastic_model(grid, so=args.so) if kname == "visco"
              else KD.elastic_model(grid, so=args.so, collocated=kname == "elastic_col"))
        dt = float(np.float32(KD.critical_dt(4.6, grid.spacing, 0.15)))
        terms = []
        for c in ("txx", "tyy", "tzz"):
            sc = KD.point_source(grid, src.coordinates, nt, 1.0, f0=0.010, name=f"src_{c}")
            terms.append(sc.inject(kd.fields[c].forward, expr=sc * S.DT))
        terms.append(rec.interpolate(kd.fields["vz"]))
    srcs = [t.sparse for t in terms if t.kind == "inject"]
    for s_ in srcs:  # Ricker sampled on this dt
        s_.data[:] = np.float32(KD.ricker(0.010, np.arange(nt) * dt, 100.0))[:, None]
    op = Operator([kd] + terms)
    mode = args.mode

    # ---- device-timed region: the native plan replays K steps ------------
    # W eager warm-up steps, GW more that capture the per-phase CUDA graphs,
    # then K timed steps (graph replay, no tracing), then the same K steps
    # again with per-action CUDA-event tracing (untimed) for the breakdown.
    plan = op._native(mode, dt)
    plan.check_cfl()  # the acoustic CFL guard (collective), once per model
    plan.run(0, args.warmup - 1)
    torch.cuda.synchronize()
    nplan = plan.plan
    stream = torch.cuda.current_stream()
    t_a = args.warmup + GW
    nplan.run(args.warmup, t_a - 1, stream)
    nplan.sync()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(ctx.device or 0)
    clocks.start()  # before the barrier: its wait for a first sample differs per rank
    # NVLink counters are read OUTSIDE the barrier-bracketed region: an NVML
    # query takes milliseconds and would skew the ranks' start times
    nvl = NvlinkCounters(ctx.device or 0) if N > 1 else None
    nv0 = nvl.read() if nvl else None
    ctx.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    nplan.run(t_a, t_a + args.steps - 1, stream)
    e1.record(stream)
    nplan.sync()
    torch.cuda.synchronize()
    clk = clocks.stop()
    ctx.barrier()
    nv1 = nvl.read() if nvl else None
    ms = e0.elapsed_time(e1)
    ms_max = ctx.allreduce_max(ms)
    # two more repetitions of the same K steps (reported, not the value):
    # run-to-run spread of the device-timed measurement
    repeats = [ms_max / args.steps]
    for _ in range(2):
        ctx.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        nplan.run(t_a, t_a + args.steps - 1, stream)
        e1.record(stream)
        nplan.sync()
        torch.cuda.synchronize()
        repeats.append(ctx.allreduce_max(e0.elapsed_time(e1)) / args.steps)
    nplan.set_tracing(True)
    ctx.barrier()
    nplan.run(t_a, t_a + args.steps - 1, stream)
    nplan.sync()
    nplan.set_tracing(False)
    rows = nplan.trace()
    launches = int(sum(r[5] for r in rows)) * args.steps

    pts_total = float(np.prod(shape))
    arr_gb = 4.0 * math.prod(grid.local_shape) / 1e9
    value = pts_total * args.steps / (ms_max * 1e-3) / 1e9

    # dominant kernel: the largest compute action (CORE in full, DOMAIN else)
    ep = plan.eplan
    comp = [(i, a) for i, a in enumerate(ep.actions) if a.kind == "compute"]
    # longest compute action of the step (per-action CUDA-event means)
    big_i, big_a = max(comp, key=lambda ia: rows[plan.native_index[ia[0]]][4])
    big_pts = math.prod(h_ - l_ for l_, h_ in zip(*big_a.box))
    big_ms = rows[plan.native_index[big_i]][4]
    kernel_label = {"acoustic": (f"star_tma<{args.so // 2}> (acoustic SO-{args.so}, TMA pipeline)"
                                 if args.so < 12 else
                                 f"star_tma2<{args.so // 2}> (acoustic SO-{args.so}, TMA pipeline, "
                                 "2 rows per thread)" if args.so < 14 else
                                 f"star_tmem<{args.so // 2}> (acoustic SO-{args.so}, TMA pipeline, "
                                 "2 rows per thread, x-window in tensor memory)"),
                    "damped": f"var-star stream kernel (acoustic + ABC layer, SO-{args.so})",
                    "rotated": (f"rot_fused (SPEC tti_gxx, SO-{args.so}, single pass)"
                                if args.so <= 8 else
                                f"rot_g + rot_update (SPEC tti_gxx, SO-{args.so})"),
                    "tti": (f"tti_fused (SO-{args.so}, single pass)" if args.so <= 6 else
                            f"tti_g + tti_update (SO-{args.so})"),
                    "elastic": f"el_velocity / el_stress (SO-{args.so})",
                    "elastic_col": f"collocated el_velocity / el_stress (SO-{args.so})",
                    "visco": f"el_velocity / visco_stress (SO-{args.so})"}[kname]
    if kname in ("elastic", "elastic_col", "visco"):
        kernel_label += f" [{big_a.kernel.kind} phase]"
    bpp = big_a.kernel.bytes_per_point
    peak, peak_src = load_peaks()
    achieved = bpp * big_pts / (big_ms * 1e-3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof):
        try:
            d = json.load(open(prof))
            key = f"{kname}_so{args.so}_{n}" if not args.shape else f"{kname}_so{args.so}_{args.shape}"
            if key in d:
                traffic = d[key].get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # ---- e2e: the public API call, host source samples in, traces out ---
    e2e = None
    try:
        ctx.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        op.apply(time_m=0, time_M=args.steps - 1, dt=dt, mpi=mode)
        el = time.perf_counter() - t0
        el = ctx.allreduce_max(el)
        e2e = {"value": pts_total * args.steps / el / 1e9, "unit": "GPts/s",
               "h2d_bytes_per_step": int(src.npoint * 4),
               "d2h_bytes_per_step": int(rec.npoint * 4),
               "how": "Operator.apply wall clock (max over ranks): src.data host->device, "
                      "rec.data device->host + gather, plan run (steady state: the "
                      "operator's CUDA graphs were captured by the untimed warm-up)"}
    except Exception as exc:  # pragma: no cover
        e2e = {"value": None, "error": str(exc)[:200]}

    # exposed halo time (N > 1): same decomposition and boxes, compute only
    exposed = None
    if N > 1:
        cplan = op._native(mode, dt, exchange=False)
        cplan.run(0, 1)
        cplan.plan.run(2, 2 + GW - 1, stream)  # graph capture, untimed
        cplan.plan.sync()
        ctx.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        cplan.plan.run(2 + GW, 2 + GW + args.steps - 1, stream)
        e1.record(stream)
        cplan.plan.sync()
        torch.cuda.synchronize()
        ms_c = ctx.allreduce_max(e0.elapsed_time(e1))
        posts = [(i, a) for i, a in enumerate(ep.actions) if a.kind == "post" and a.messages]
        sent = sum(m.volume * sum(a.spot.sends(f, t, m.direction) for f, t in a.spot.fields)
                   for _i, a in posts for m in a.messages) * 4
        post_ms = sum(rows[plan.native_index[i]][4] for i, _a in posts)
        fused = any(a.pushed for _i, a in posts)
        if fused:
            # halos travel inside the OWNED-slab kernels (peer stores); the
            # post only releases flags, so report the slab kernels' time
            slabs = [i for i, a in enumerate(ep.actions)
                     if a.kind == "compute" and a.region == "OWNED"]
            post_ms = sum(rows[plan.native_index[i]][4] for i in slabs)
        exposed = {"exposed_ms_per_step": (ms_max - ms_c) / args.steps,
                   "step_ms": ms_max / args.steps, "compute_only_step_ms": ms_c / args.steps,
                   "exposed_frac": (ms_max - ms_c) / ms_max,
                   "halo_bytes_sent_per_step_rank0": sent,
                   "transport": ("fused: OWNED-slab kernels store into peer halos (NVLink)"
                                 if fused else "copy engines (cudaMemcpy3DAsync, 4 streams)"),
                   "post_ms_rank0": post_ms,
                   # fused: bytes pushed / time of the slab kernels that push them
                   # (a lower bound on the link rate: the stores are spread
                   # over the slabs' compute)
                   "link_gbs_rank0": (sent / (post_ms * 1e-3) / 1e9 if post_ms > 0 else None),
                   "link_peak_gbs": 900.0}
        if fused:
            exposed["link_note"] = ("halos are stored by the OWNED-slab kernels while they "
                                    "compute (no separate transfer to time); post_ms_rank0 is "
                                    "the slab kernels' time, the exposed time is the cost")
        if not (nv0 and nv1):
            exposed["nvlink_counters_rank0"] = ("unavailable: NVML reports the NVLink data "
                                                "counters as not supported on this box")
        if nv0 and nv1:
            # NVML NVLink data counters over the timed region (rank 0's GPU)
            tx = (nv1["tx"] - nv0["tx"]) / args.steps
            rx = (nv1["rx"] - nv0["rx"]) / args.steps
            exposed["nvlink_counters_rank0"] = {
                "tx_bytes_per_step": tx, "rx_bytes_per_step": rx,
                "tx_gbs_step_avg": tx / (ms_max / args.steps * 1e-3) / 1e9,
                "tx_gbs_during_transfer": (tx / (post_ms * 1e-3) / 1e9) if post_ms > 0 else None,
                "transfer_window": ("OWNED-slab kernels (fused push)" if fused
                                    else "copy-engine posts"),
                "peak_gbs_per_direction": 900.0,
                "source": "NVML NVLINK_THROUGHPUT_DATA_TX/RX, summed over links"}


    # per-rank action timings (skew between ranks shows up as WAIT time)
    rank_actions = ctx.allgather([[int(r[2]), round(r[4], 4)] for r in rows]) if N > 1 else None

    cpu = None
    if ctx.rank == 0 and N == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_reference(n, args.so, args.cpu_seconds)
        except Exception as exc:  # pragma: no cover
            cpu = {"error": str(exc)[:200]}

    if ctx.rank == 0:
        line = {
            "metric": "GPts/s", "value": value, "unit": "GPts/s", "n_gpus": N,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True,
            "scaling": "strong" if args.shape and N > 1 else "weak", "vs_baseline": None, "dtype": "fp32",
            "data": "synthetic (layered vp + hashed noise, Ricker source, receiver line)",
            "config": {"workload": (f"3D isotropic acoustic SO-{args.so}, {n}^3 per GPU "
                                    "(BASELINE configs[1])") if kname == "acoustic" and not args.shape
                       else f"3D {kname} SO-{args.so}, global {shape}",
                       "global_shape": list(shape), "topology": list(topo), "mode": mode,
                       "parallelism": f"domain decomposition x/y {topo}",
                       "sources": 1, "receivers": args.nrec,
                       "untimed_steps": f"{args.warmup} warm-up + {GW} graph-capture",
                       "l2": f"no flush: every array ({arr_gb:.1f} GB per rank) >> 126 MB L2"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": kernel_label,
                         "bytes_per_point": bpp, "points_per_launch": big_pts,
                         "launch_ms": big_ms, "peak_source": peak_src},
            "gpu_launches": launches,
            "repeat_ms_per_step": [round(r, 4) for r in repeats],
            "e2e": e2e,
            "clocks": clk,
            "halo": exposed,
            "cpu_baseline": cpu,
            "step_actions": [{"kind": int(r[2]), "stream": int(r[1]),
                              "ms": round(r[4], 4)} for r in rows],
            "rank_actions": rank_actions,
        }
        print(json.dumps(line), flush=True)
    ctx.barrier()
    # release the plans (IPC mappings, streams, graphs) before the process
    # group goes away, then exit normally
    del op, plan, nplan
    import gc
    gc.collect()
    torch.cuda.synchronize()
    ctx.barrier()
    if world > 1 and dist.is_initialized():
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    rc = main()
    sys.stdout.flush()
    sys.exit(rc or 0)
