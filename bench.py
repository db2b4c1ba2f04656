"""Benchmark of the B200 hot path: FMG + error estimator on the HHG (arXiv 2508.06049).

Contract (driver): ``python bench.py --gpus N --steps K --warmup W [--impl reference]``
prints ONE JSON line on rank 0.

Workload (BASELINE.json configs[1], "config 2"): the 2-D L-shaped domain, P1
fp64, L = 7 structured levels, FMG with nu = 2 V(2,2)-cycles per level and the
j = 1 error estimate, over the six coarse meshes T_0^k, k = 0..5, of the 5-step
kl AMR run (estimate -> mark >= 0.5 max -> refine -> re-solve); the meshes are
the ones the patched reference itself produces (tests/golden/cfg2_k*.mesh).
One step = fmg() + error_estimate(j=1) on each of the six hierarchies in AMR
order (the hot path of run_kl, proj/src/amr.cpp:176-213); hierarchy build and
upload happen once, outside the timed region, as SURVEY.md §8(d) specifies.

value     = unique fine DoF of the step / device time of the step, GDoF/s,
            inputs resident in HBM, L2 flushed between steps (256 MiB write).
e2e       = the same through the public API with host buffers: per mesh
            set_problem (host tabulation + pinned H2D), fmg(), error_estimate()
            (eta_T to the host) and u_L read back to pinned host memory.
roofline  = the dominant kernel (by device time) from CUDA-event probes inside
            the timed region: algorithmic bytes / its time,
            against MEASURED_PEAKS.json's copy bandwidth.
cpu_baseline = the patched reference (oracle/_ref/ref_driver, compiled from
            /root/reference sources) on one host core, a bounded sample.
--impl reference = the same reference, single-threaded as it is written (one
            solve cannot use more threads); the all-cores replica aggregate is
            reported beside it for context.
Multi-GPU: the 2-D parity path does not shard (exact Gauss-Seidel order,
SURVEY.md §8(e)): N ranks run N independent replicas ("scaling": "weak").
The 3-d configuration 5 does shard: at N > 1 its macros are split over the
ranks (NCCL interface exchange; workloads_3d.cfg5_sharded, strong scaling).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

MESH_DIR = os.path.join(REPO, "tests", "golden")
CFG2_MESHES = [f"cfg2_k{k}.mesh" for k in range(6)]
LEVEL = 7
NU = 2
METRIC = "FMG+estimator DoF throughput (cfg2 L-shape AMR meshes, l=7, V(2,2) nu=2)"
UNIT = "GDoF/s"
REF_DRIVER = os.path.join(REPO, "oracle", "_ref", "ref_driver")
FLUSH_BYTES = 256 << 20
SHARDED_TIMEOUT_S = 300  # watchdog of the NCCL-sharded secondary run


def peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------- reference arm (CPU)
def run_reference_driver(steps, warmup, procs=1):
    """Run `procs` concurrent single-threaded reference processes; returns their JSON records."""
    cmd = [REF_DRIVER, "timeall", "lshape", str(LEVEL), str(NU), str(steps), str(warmup)] + CFG2_MESHES
    ps = [subprocess.Popen(cmd, cwd=MESH_DIR, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
          for _ in range(procs)]
    out = []
    for p in ps:
        so, se = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"ref_driver failed: {se.strip()[-400:]}")
        out.append(json.loads(so.strip().splitlines()[-1]))
    return out


def cpu_port_sample(steps):
    """Fallback CPU baseline when the reference binary is absent: the C restatement oracle."""
    from oracle import oracle as O
    from paper_2508_06049_b200 import klref as K

    meshes = [K.MacroMesh.read(os.path.join(MESH_DIR, m)) for m in CFG2_MESHES]
    hs = [O.Hier2D(m, LEVEL) for m in meshes]
    dofs = sum(h.dofs(LEVEL) for h in hs)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        for m, h in zip(meshes, hs):
            st = O.fmg2d(m, LEVEL, problem="lshape", nu=NU, hier=h)
            O.estimate2d(st, 1)
        times.append(time.perf_counter() - t0)
    return dofs, times


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def impl_reference(args):
    """The reference's own CPU implementation of the path (the patched reference
    compiled from /root/reference sources, oracle/_ref/ref_driver).  The
    reference is single-threaded (no threads, no MPI), so one
    solve uses exactly one host thread -- that is the reference arm.  For
    context the line also carries the aggregate of one independent replica per
    host core (`replicas_all_cores`), the throughput a box full of separate AMR
    runs would reach."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cores = host_cores()
    replicas = None
    if os.path.exists(REF_DRIVER):
        rec = run_reference_driver(args.steps, args.warmup, procs=1)[0]
        dofs = rec["dofs_per_step"]
        t = statistics.mean(rec["step_s"])
        value = dofs / t / 1e9
        ms = t * 1e3
        kind = "reference"
        sample = (f"patched reference (oracle/_ref/ref_driver, g++ -O2), single-threaded like the reference, "
                  f"{args.steps} full steps after {args.warmup} warm-up")
        if not args.no_replicas and cores > 1:
            recs = run_reference_driver(max(1, min(args.steps, 3)), 1, procs=cores)
            per_proc = [statistics.mean(r["step_s"]) for r in recs]
            replicas = {"value": sum(dofs / tt for tt in per_proc) / 1e9, "unit": UNIT, "processes": cores,
                        "note": "one independent single-threaded replica per host core (context, not the arm)"}
    else:
        dofs, times = cpu_port_sample(args.steps)
        value = dofs / statistics.mean(times) / 1e9
        ms = statistics.mean(times) * 1e3
        kind = "port"
        sample = f"C restatement oracle, {args.steps} full steps, 1 thread (reference binary absent)"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(dofs),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": kind, "sample": sample,
                             "host_cores": cores, "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "replicas_all_cores": replicas}
    print(json.dumps(line), flush=True)
    return 0


def workload_config(dofs):
    return {"workload": "cfg2: L-shape (-1,1)^2\\[0,1)x(-1,0], 6 macro triangles -> 5 kl AMR steps "
                        "(meshes k=0..5), l=7, P1 fp64, FMG V(2,2) nu=2 + estimator j=1 per mesh",
            "meshes": CFG2_MESHES, "level": LEVEL, "nu": NU, "dofs_per_step": dofs,
            "l2": "flushed between timed steps (256 MiB write)", "parallelism": "replicas"}


# ----------------------------------------------------------------- 3-d workloads (secondary)
# BASELINE.json configs 3 and 5 (the reference has no 3-d solver: the path is
# the builder's design, pinned to the 3-d C oracle).  Reported in
# the same JSON line, not as the headline.
def fmg_bytes_3d(dofs_L, nu):
    """Algorithmic FMG bytes: (190.7 nu + 28.6) N_L (3-d)."""
    return (190.7 * nu + 28.6) * dofs_L


def run_3d(K, torch, name, N, L, prob, reps, peak):
    from paper_2508_06049_b200.meshes import kuhn_cube, series_coefficients

    t0 = time.perf_counter()
    h = K.GridHierarchy.build(kuhn_cube(N), L)
    kind = {"sin3": K.PROBLEM_SIN3D, "series": K.PROBLEM_SERIES3D}[prob]
    s = K.MultigridSolver(h, K.Problem(kind, series_coefficients() if prob == "series" else None),
                          K.SolverConfig(nu=2))
    build_s = time.perf_counter() - t0
    stream = torch.cuda.ExternalStream(s.stream())
    s.set_profiling(True)
    s.fmg_enqueue()
    s.error_estimate_enqueue(1)
    s.synchronize()
    s.error_estimate_finish(1, K.UNSCALED)
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    times, kms, kb = [], [0.0] * 8, [0.0] * 8
    for it in range(reps):
        with torch.cuda.stream(stream):
            flush.fill_(float(it))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        s.fmg_enqueue()
        s.error_estimate_enqueue(1)
        e1.record(stream)
        s.synchronize()
        rep = s.error_estimate_finish(1, K.UNSCALED)
        times.append(e0.elapsed_time(e1))
        for kk in range(8):
            m_, _, b_ = s.kernel_stats(kk)
            kms[kk] += m_
            kb[kk] += b_
    ms = sum(times) / len(times)
    dofs = h.dof_count(L)
    est_ms = kms[K.KERNEL_ESTIMATE] / reps
    gs_gbs = kb[K.KERNEL_GS] / (kms[K.KERNEL_GS] * 1e-3) / 1e9 if kms[K.KERNEL_GS] > 0 else None
    fmg_ms = ms - est_ms
    # headline-shaped roofline of this workload's dominant kernel (CUDA-event
    # probes in the captured graph, algorithmic bytes of SURVEY.md §8(d))
    dom = max(range(8), key=lambda k: kms[k])
    n_dom = s.kernel_stats(dom)[1]
    ach = kb[dom] / (kms[dom] * 1e-3) / 1e9 if kms[dom] > 0 else 0.0
    traffic = None
    try:
        with open(os.path.join(REPO, "profiles", "ncu_traffic.json")) as fh:
            traffic = json.load(fh).get(f"{name.split(':')[0]}_{K.KERNEL_NAMES[dom]}")
    except Exception:
        traffic = None
    roof = {"bound": "hbm", "kernel": K.KERNEL_NAMES[dom], "achieved": ach, "peak": peak, "unit": "GB/s",
            "frac": ach / peak, "traffic": traffic, "alg_bytes_per_launch": kb[dom] / reps / max(n_dom, 1),
            "ms_per_launch": kms[dom] / reps / max(n_dom, 1), "launches_per_fmg": n_dom}
    return {"config": name, "mesh": f"Kuhn {N}^3 cubes x 6 tets ({h.num_macros()} macros)", "level": L,
            "dofs": dofs, "ms_fmg_plus_estimate": ms, "estimator_ms": est_ms, "value": dofs / (ms * 1e-3) / 1e9,
            "unit": "GDoF/s", "fmg_roofline": {"alg_bytes": fmg_bytes_3d(dofs, 2),
                                               "frac": fmg_bytes_3d(dofs, 2) / (fmg_ms * 1e-3) / 1e9 / peak},
            "roofline": roof, "smoother_alg_GBps": gs_gbs, "eta": rep.eta, "theta": rep.conv_factor,
            "kernel_ms": {K.KERNEL_NAMES[k]: kms[k] / reps for k in range(8) if kms[k] > 0},
            "build_s": build_s, "parity": "builder 3-d oracle (oracle/klref_oracle3d.c), bitwise on small cases"}


def run_kl_loop():
    """BASELINE.json config 2 end to end through the product: the 5-step kl
    loop of build/dropin/dropin_kl (the reference's own mesh layer linked
    against the facade; per step host hierarchy build + upload, FMG, estimate,
    >= 0.5 max marks, refine_rg), wall clock of the whole loop."""
    exe = os.path.join(REPO, "build", "dropin", "dropin_kl")
    if not os.path.exists(exe):
        return {"error": "build/dropin/dropin_kl not built (needs the reference sources at build time)"}
    import tempfile
    with tempfile.TemporaryDirectory() as tmp:
        runs = []
        for _ in range(2):  # the second run is reported (first-touch of the library and device)
            r = subprocess.run([exe, "halfmax", os.path.join(MESH_DIR, CFG2_MESHES[0]), "lshape", "5", str(LEVEL),
                                str(NU), tmp], capture_output=True, text=True, timeout=600)
            if r.returncode != 0:
                return {"error": r.stderr.strip()[-300:]}
            lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
            runs.append(lines)
    steps = [d for d in runs[-1] if "k" in d]
    tail = runs[-1][-1]
    dofs = sum(d["dofs"] for d in steps)
    return {"workload": "cfg2 kl loop: k = 0..5, build + upload + FMG + estimate + mark + refine per step "
                        "(the process's CUDA context is created before the loop and reported as device_init_seconds)",
            "loop_seconds": tail["loop_seconds"], "build_solve_estimate_seconds": tail["build_solve_estimate_seconds"],
            "device_init_seconds": tail.get("device_init_seconds"),
            "hierarchy_seconds": tail.get("hierarchy_seconds"),
            "hierarchy_solver_build_seconds": tail.get("hierarchy_solver_build_seconds"),
            "fmg_seconds": tail.get("fmg_seconds"), "estimate_seconds": tail.get("estimate_seconds"),
            "dofs": dofs, "value": dofs / tail["loop_seconds"] / 1e9, "unit": "GDoF/s",
            "macros": [d["macros"] for d in steps], "marks": [d["marks"] for d in steps[:-1]],
            "eta": [d["eta"] for d in steps]}


def run_cfg4(K, torch, reps, peak):
    """Config 4: the 3-d AMR sequence (tests/golden/cfg4_k*.mesh, the reference's
    refine_rg_3d driven by the 3-d oracle): one step = FMG + estimate + the
    >= 0.5 max marks on each of the five meshes, device time."""
    with open(os.path.join(MESH_DIR, "cfg4.json")) as fh:
        meta = json.load(fh)
    L = meta["level"]
    hs, solvers = [], []
    for k in range(len(meta["steps"])):
        h = K.GridHierarchy.build(K.MacroMesh.read(os.path.join(MESH_DIR, f"cfg4_k{k}.mesh")), L)
        hs.append(h)
        solvers.append(K.MultigridSolver(h, K.Problem(K.PROBLEM_GAUSS3D), K.SolverConfig(nu=meta["nu"])))
    stream = torch.cuda.Stream()
    for s in solvers:
        s.set_stream(stream.cuda_stream)
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")

    def step():
        marks_ok = True
        for s in solvers:
            s.fmg_enqueue()
            s.error_estimate_enqueue(1)
        for k, s in enumerate(solvers):
            s.synchronize()
            rep = s.error_estimate_finish(1, K.UNSCALED)
            st = meta["steps"][k]
            if "marks_halfmax_eta" in st:
                marks_ok &= K.mark(K.MARK_HALF_MAX, 0.0, st["active_ids"], st["green_parent"], rep.eta_local,
                                   st["reverted_ids"]) == st["marks_halfmax_eta"]
        return marks_ok

    step()
    times, ok = [], True
    for it in range(reps):
        with torch.cuda.stream(stream):
            flush.fill_(float(it))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for s in solvers:
            s.fmg_enqueue()
            s.error_estimate_enqueue(1)
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
        ok &= step()
    ms = sum(times) / len(times)
    dofs = sum(h.dof_count(L) for h in hs)
    return {"config": "cfg4: unit cube, 6 Kuhn tets -> 4 kl AMR steps (meshes k=0..4), l=6, Gaussian peak, "
                      "FMG V(2,2) + estimator per mesh", "macros": [h.num_macros() for h in hs], "level": L,
            "dofs": dofs, "ms_fmg_plus_estimate": ms, "value": dofs / (ms * 1e-3) / 1e9, "unit": "GDoF/s",
            "fmg_roofline": {"alg_bytes": fmg_bytes_3d(dofs, meta["nu"]),
                             "frac": fmg_bytes_3d(dofs, meta["nu"]) / (ms * 1e-3) / 1e9 / peak},
            "marks_equal_fixture": bool(ok),
            "parity": "eta_T within 1e-9 and identical marks vs the 3-d oracle fixtures (tests/test_cfg4_3d.py)"}


def run_3d_sharded(K, torch, dist, world, rank, reps, peak, barrier, max_over_ranks):
    """Config 5 strong scaling: the 3072 macro tets sharded over the `world`
    GPUs (contiguous slot ranges = z-slabs), interface exchange over NCCL,
    levels <= 3 replicated.  All ranks call this; rank 0 reports."""
    from paper_2508_06049_b200.meshes import kuhn_cube, series_coefficients

    L = 6
    t0 = time.perf_counter()
    h = K.GridHierarchy.build(kuhn_cube(8), L)
    uid = [K.Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    # NCCL announces its version on stdout at init: keep stdout for the JSON line
    sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)
    try:
        comm = K.Comm(world, rank, uid[0])
    finally:
        os.dup2(saved, 1)
        os.close(saved)
    prob = K.Problem(K.PROBLEM_SERIES3D, series_coefficients())
    s = K.ShardedSolver(h, prob, K.SolverConfig(nu=2), comm=comm, rep_level=3)
    build_s = time.perf_counter() - t0
    stream = torch.cuda.ExternalStream(s.stream())
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    for _ in range(2):
        s.fmg_enqueue()
        s.error_estimate_enqueue(1)
        s.synchronize()
        rep = s.error_estimate_finish(1, K.UNSCALED)
    times = []
    for it in range(reps):
        with torch.cuda.stream(stream):
            flush.fill_(float(it))
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        s.fmg_enqueue()
        s.error_estimate_enqueue(1)
        e1.record(stream)
        s.synchronize()
        rep = s.error_estimate_finish(1, K.UNSCALED)
        times.append(e0.elapsed_time(e1))
    ms = max_over_ranks(sum(times) / len(times))
    fl, el, xb = s.counts()
    dofs = h.dof_count(L)
    s.close()
    comm.close()
    return {"config": "cfg5: unit cube, 8^3 Kuhn cubes, l=6, sine series (g=0), macros sharded over the GPUs",
            "n_gpus": world, "scaling": "strong", "dofs": dofs, "ms_fmg_plus_estimate": ms,
            "value": dofs / (ms * 1e-3) / 1e9, "unit": "GDoF/s",
            "fmg_roofline_aggregate": {"alg_bytes": fmg_bytes_3d(dofs, 2),
                                       "frac": fmg_bytes_3d(dofs, 2) / (ms * 1e-3) / 1e9 / (peak * world)},
            "exchange_bytes_per_fmg_rank0": xb, "launches_per_fmg_rank0": fl, "eta": rep.eta,
            "theta": rep.conv_factor, "build_s": build_s, "rep_level": 3,
            "parity": "bitwise equal to the one-device solver (tests/test_shard_3d.py, in-process shards)"}


def cpu_3d_port_sample(level=6):
    """Single-threaded 3-d C oracle on config 3 itself (4^3 Kuhn cubes, l = 6,
    17 M DoF): one FMG + estimate (about 30 s of CPU work)."""
    from oracle import oracle as O
    from paper_2508_06049_b200.meshes import kuhn_cube

    m = kuhn_cube(4)
    h = O.Hier3D(m.coords, m.elements, level)
    t0 = time.perf_counter()
    st = O.fmg3d(h, "sin3", nu=2)
    O.estimate3d(st)
    dt = time.perf_counter() - t0
    return {"value": h.dofs(level) / dt / 1e9, "unit": "GDoF/s", "cores": 1, "kind": "port",
            "ms_fmg_plus_estimate": dt * 1e3, "host_cores": host_cores(), "cpu_model": cpu_model(),
            "sample": f"3-d C oracle (builder restatement, not the reference: the reference has no 3-d solver), "
                      f"config 3 at l={level} ({h.dofs(level)} DoF), one FMG + estimate, 1 thread"}


# ----------------------------------------------------------------- our arm (GPU)
def impl_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2508_06049_b200 import klref as K

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (the hot path has no CPU fallback)")
    torch.cuda.set_device(local)
    if world > 1 or args.force_sharded_3d:
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    K.lib()

    meshes = [K.MacroMesh.read(os.path.join(MESH_DIR, m)) for m in CFG2_MESHES]
    hs = [K.GridHierarchy.build(m, LEVEL) for m in meshes]
    problem = K.Problem(K.PROBLEM_LSHAPE)
    solvers = [K.MultigridSolver(h, problem, K.SolverConfig(nu=NU, use_graph=1)) for h in hs]
    dofs = sum(h.dof_count(LEVEL) for h in hs)
    stream = torch.cuda.Stream()
    for s in solvers:
        s.set_stream(stream.cuda_stream)
        s.set_profiling(True)
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")

    def enqueue_step():
        for s in solvers:
            s.fmg_enqueue()
            s.error_estimate_enqueue(1)

    def finish_step():
        for s in solvers:
            s.synchronize()  # raises SolverError if a level-0 CG failed
            s.error_estimate_finish(1, K.UNSCALED)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # warm-up (graph capture happens here)
    for _ in range(max(args.warmup, 0)):
        enqueue_step()
        finish_step()
    launches_per_step = sum(s.launch_count() + s.estimate_launch_count() for s in solvers)

    nkinds = 8
    kern_ms = [0.0] * nkinds
    kern_bytes = [0.0] * nkinds
    kern_n = [0] * nkinds
    step_ms = []
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    for it in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(float(it))
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        enqueue_step()
        ev1.record(stream)
        finish_step()
        step_ms.append(ev0.elapsed_time(ev1))
        for kind in range(nkinds):
            ms = b = 0.0
            n = 0
            for s in solvers:
                m_, n_, b_ = s.kernel_stats(kind)
                ms += m_
                n += n_
                b += b_
            kern_ms[kind] += ms
            kern_bytes[kind] += b
            kern_n[kind] += n
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    t_step = max_over_ranks(sum(step_ms) / len(step_ms))

    # ---- end to end through the public API with host buffers
    u_host = [torch.empty(h.level_size(LEVEL), dtype=torch.float64, pin_memory=True).numpy() for h in hs]
    e2e_ms = []
    h2d = d2h = 0
    barrier()
    torch.cuda.synchronize()
    for it in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(float(it))
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        hb = db = 0
        for s, h, uh in zip(solvers, hs, u_host):
            hb += s.set_problem(problem)
            s.fmg()
            rep = s.error_estimate(1, K.UNSCALED)
            s.state_into(K.STATE_U, LEVEL, uh)
            db += uh.nbytes + 2 * 8 * h.num_macros() + 16
        ev1.record(stream)
        ev1.synchronize()
        e2e_ms.append(ev0.elapsed_time(ev1))
        h2d, d2h = hb, db
    torch.cuda.synchronize()
    barrier()
    t_e2e = max_over_ranks(sum(e2e_ms) / len(e2e_ms))
    _ = rep

    sharded = (world > 1 or args.force_sharded_3d) and not args.no_3d
    if rank != 0:
        if sharded:
            try:
                run_3d_sharded(K, torch, dist, world, rank, 3, peaks()[0], barrier, max_over_ranks)
            except Exception:
                pass
        if dist.is_initialized():
            dist.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel (largest device time in the probes)
    peak, peak_src = peaks()
    dom = max(range(nkinds), key=lambda k: kern_ms[k])
    ach = kern_bytes[dom] / (kern_ms[dom] * 1e-3) / 1e9 if kern_ms[dom] > 0 else 0.0
    traffic = None
    tpath = os.path.join(REPO, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as fh:
                traffic = json.load(fh).get(K.KERNEL_NAMES[dom])
        except Exception:
            traffic = None
    breakdown = {}
    probe_total = sum(kern_ms)
    for k in range(nkinds):
        if kern_n[k] == 0:
            continue
        breakdown[K.KERNEL_NAMES[k]] = {
            "ms_per_step": kern_ms[k] / args.steps, "launches_per_step": kern_n[k] / args.steps,
            "alg_GBps": (kern_bytes[k] / (kern_ms[k] * 1e-3) / 1e9) if kern_ms[k] > 0 else None,
            "share": kern_ms[k] / probe_total if probe_total > 0 else None}
    est_ms = kern_ms[K.KERNEL_ESTIMATE] / args.steps

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            if os.path.exists(REF_DRIVER):
                rec = run_reference_driver(args.cpu_steps, 1, procs=1)[0]
                cv = rec["dofs_per_step"] / statistics.mean(rec["step_s"]) / 1e9
                cpu = {"value": cv, "unit": UNIT, "cores": 1, "kind": "reference",
                       "sample": f"{args.cpu_steps} full steps (6 meshes x FMG + estimate) of the patched reference "
                                 f"(oracle/_ref/ref_driver, g++ -O2, single-threaded), after 1 warm-up",
                       "ms_per_step": statistics.mean(rec["step_s"]) * 1e3, "host_cores": host_cores(),
                       "cpu_model": cpu_model()}
            else:
                cd, ct = cpu_port_sample(max(1, args.cpu_steps // 2))
                cpu = {"value": cd / statistics.mean(ct) / 1e9, "unit": UNIT, "cores": 1, "kind": "port",
                       "sample": f"{len(ct)} full steps of the C restatement oracle, single-threaded",
                       "ms_per_step": statistics.mean(ct) * 1e3}
        except Exception as exc:  # the baseline is reported, not required
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference", "sample": f"failed: {exc}"}

    extra3d = None
    if sharded:
        extra3d = {"cfg5_sharded": None}  # filled after the headline line is ready (below)
    elif not args.no_3d:
        try:
            peak3, _ = peaks()
            extra3d = {"cfg3": run_3d(K, torch, "cfg3: unit cube, 4^3 Kuhn cubes, l=6, sin3", 4, 6, "sin3", 3, peak3),
                       "cfg4": run_cfg4(K, torch, 3, peak3),
                       "cfg5_one_gpu": run_3d(K, torch, "cfg5: unit cube, 8^3 Kuhn cubes, l=6, sine series (g=0)",
                                              8, 6, "series", 2, peak3)}
            if world == 1 and not args.no_cpu_baseline:
                extra3d["cpu_baseline_3d"] = cpu_3d_port_sample()
        except Exception as exc:  # secondary numbers never sink the headline line
            extra3d = {"error": str(exc)[:300]}
    kl_loop = None
    if world == 1 and not args.no_3d:
        try:
            kl_loop = run_kl_loop()
        except Exception as exc:  # secondary numbers never sink the headline line
            kl_loop = {"error": str(exc)[:300]}

    value = world * dofs / (t_step * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(dofs),
        "fmg_ms_per_step": t_step - est_ms, "estimator_ms_per_step": est_ms,
        "roofline": {"bound": "hbm", "kernel": K.KERNEL_NAMES[dom], "achieved": ach, "peak": peak,
                     "peak_source": peak_src, "unit": "GB/s", "frac": ach / peak, "traffic": traffic,
                     "alg_bytes_per_launch": kern_bytes[dom] / max(kern_n[dom], 1),
                     "ms_per_launch": kern_ms[dom] / max(kern_n[dom], 1)},
        "kernels": breakdown,
        "e2e": {"value": world * dofs / (t_e2e * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": t_e2e,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk,
        "cpu_baseline": cpu,
        "workloads_3d": extra3d,
        "kl_loop_e2e": kl_loop,
    }
    if sharded:
        # the NCCL-sharded config-5 run (all ranks): a watchdog prints the
        # headline line without it and ends the job if it does not finish
        done = threading.Event()
        printed = threading.Lock()

        def watchdog():
            if not done.wait(SHARDED_TIMEOUT_S):
                with printed:
                    extra3d["cfg5_sharded"] = {"error": f"timed out after {SHARDED_TIMEOUT_S} s"}
                    print(json.dumps(line), flush=True)
                    os._exit(0)

        threading.Thread(target=watchdog, daemon=True).start()
        try:
            res = run_3d_sharded(K, torch, dist, world, rank, 3, peaks()[0], barrier, max_over_ranks)
        except Exception as exc:  # secondary numbers never sink the headline line
            res = {"error": str(exc)[:300]}
        with printed:
            done.set()
            extra3d["cfg5_sharded"] = res
            print(json.dumps(line), flush=True)
    else:
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-steps", type=int, default=12, help="steps of the single-core reference sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-3d", action="store_true", help="skip the secondary 3-d workloads (configs 3 and 5)")
    ap.add_argument("--force-sharded-3d", action="store_true",
                    help="run the NCCL-sharded config-5 path even at N = 1 (plumbing check)")
    ap.add_argument("--no-replicas", action="store_true", help="reference arm: skip the all-cores replica context run")
    args = ap.parse_args()
    if args.impl == "reference":
        return impl_reference(args)
    return impl_ours(args)


if __name__ == "__main__":
    sys.exit(main())
