#!/usr/bin/env python
"""femforge-b200 benchmark: assembled elements/sec (+ HBM GB/s) of the numeric
FE assembly -- K0 zero-fill + K2 element kernel with CSR/RHS scatter into a
prebuilt pattern (the reference's criterion-9 protocol, acceptance.cpp:292-327)
-- on the BASELINE.json north-star workload: 3D P2 Poisson on the Kuhn 128^3
cube (12,582,912 tets, 16,974,593 DOFs, 484,609,025 nnz).

  python bench.py [--gpus N --steps K --warmup W] [--config ns|c1|c2|c3|c4]
  torchrun --nproc-per-node N bench.py --gpus N ...   (strong scaling: row blocks of the one mesh;
                                                       --scaling weak: one cell per GPU)
  python bench.py --impl reference ...                (reference CPU arm)

One JSON line on rank 0. Multi-GPU: contiguous DOF row blocks, halo elements
duplicated, no collective on the data path; the NCCL process
group only provides the barrier and the max-over-ranks of the timings.
"""
import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "ns": dict(dim=3, degree=2, n=128, form="poisson", quad=4,
               workload="3D P2 Poisson tets, Kuhn 128^3 cube (north star, BASELINE.json)"),
    "c1": dict(dim=2, degree=1, n=512, form="poisson", quad=3,
               workload="2D P1 Poisson triangles, unit square 512x512 (BASELINE.json config 1)"),
    "c2": dict(dim=3, degree=1, n=128, form="poisson", quad=4,
               workload="3D P1 Poisson tets, Kuhn 128^3 cube (BASELINE.json config 2)"),
    "c3": dict(dim=3, degree=2, n=96, form="poisson", quad=4,
               workload="3D P2 Poisson tets, Kuhn 96^3 cube, stiffness + load (BASELINE.json config 3)"),
    "c4": dict(dim=3, degree=2, n=96, form="varcoef", quad=14,
               workload="3D P2 var-coef mass+stiffness+convection, Kuhn 96^3, 14-point rule (config 4)"),
    "c5": dict(dim=3, degree=2, n=160, form="elasticity", quad=4, ncomp=3,
               workload="3D vector P2 linear elasticity (lam=mu=1, f=(0,0,-1)), Kuhn 160^3, row blocks (config 5)"),
}
METRIC = "assembled elements/sec (3D P2 Poisson tets)"
STEP_DESC = {
    "atomic": "K0 zero-fill + K2 element kernel with fp64-RED scatter",
    "gather": "K2a element invariants + K2b row gather (class-specialised + generic; atomic-free, each CSR value "
              "written once, no zero-fill), one ff_assemble_device call per step (replayed CUDA graph); "
              "k2a_ms / k2_ms from a separate phase-split run",
}
KERNEL_DESC = {
    "atomic": "ff_assemble_atomic (K2)",
    "gather": "ff_gather_invariants + ff_gather_classes_s/_l + ff_gather_rows (K2a + K2b, the whole step)",
}
UNIT = "elements/s"


def make_mesh(ff, cfg):
    if cfg["dim"] == 2:
        coords, vconn = ff.unit_square_mesh(cfg["n"])
        dconn, n_dofs = (vconn, coords.shape[0]) if cfg["degree"] == 1 else ff.p2_dofs(2, vconn, coords.shape[0])
    else:
        coords, vconn = ff.kuhn_mesh(cfg["n"])
        dconn, n_dofs = (vconn, coords.shape[0]) if cfg["degree"] == 1 else ff.kuhn_p2_dofs(cfg["n"], vconn)
    return coords, vconn, dconn, n_dofs


def workload_config(cfg, world, elements, dofs, nnz, weak=False):
    """The `config` object of the JSON line: the workload only (mesh, form,
    sizes, partitioning), identical in both arms; diagnostics go to `detail`."""
    values_bytes = nnz * 8
    return {"workload": cfg["workload"] + (f", stacked x{world} along the last axis (one cell per GPU)"
                                           if weak else ""),
            "n": cfg["n"], "elements": int(elements), "dofs": int(dofs), "nnz": int(nnz), "form": cfg["form"],
            "quad_rule": cfg["quad"],
            "parallelism": f"row-blocks x{world} (halo elements duplicated, no collective)",
            "l2": "flushed (256 MiB write) between steps" if values_bytes < 2 * 126 * 2 ** 20 else
                  f"inputs > L2 (CSR values {values_bytes / 1e9:.2f} GB)"}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def fp64_peak():
    """Measured fp64 FMA peak (tools/microbench/fp64_peak.cu on a B200,
    profiles/r2_fp64_peak.json), else the nominal 37 TFLOP/s."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2_fp64_peak.json")) as f:
            return float(json.load(f)["fp64_tflops"]), "measured (profiles/r2_fp64_peak.json, DFMA microbench)"
    except Exception:
        return 37.0, "nominal B200 fp64"


FP64_PEAK_TFLOPS, FP64_PEAK_SOURCE = fp64_peak()


def model_flops(cfg):
    """SURVEY.md §8d flop model per element: geometry 60; per quadrature point
    n_local*15 (basis gradients) + entries * (7 stiffness | +3 mass | +7
    convection) + load 25 + 2 n_local. Reference-tensor forms (quadrature
    summed at compile time) are quoted with their symmetric count."""
    k = {(2, 1): 3, (2, 2): 6, (3, 1): 4, (3, 2): 10}[(cfg["dim"], cfg["degree"])]
    nq = {1: 1, 3: 3, 4: 4, 11: 11, 14: 14}.get(cfg["quad"], cfg["quad"])
    if cfg["form"] == "elasticity":   # §8d C5: vector P2, 465 symmetric entries of the 30x30 element matrix
        kk = 3 * k
        return 60 + nq * (k * 15 + kk * (kk + 1) // 2 * 7 + 25 + 2 * kk)
    per_entry = {"poisson": 7, "stiffness": 7, "mass": 3, "helmholtz": 10, "demo2d": 10, "varcoef": 17}[cfg["form"]]
    entries = k * (k + 1) // 2 if cfg["form"] != "varcoef" else k * k
    return 60 + nq * (k * 15 + entries * per_entry + 25 + 2 * k)


def algorithmic_bytes(cfg, n_elems, n_vertices, n_rows, nnz):
    """SURVEY.md §8d compulsory-traffic model: connectivity + coordinates +
    CSR values written and col_idx read + row_ptr + RHS."""
    k = {(2, 1): 3, (2, 2): 6, (3, 1): 4, (3, 2): 10}[(cfg["dim"], cfg["degree"])]
    w_rp = 8 if nnz >= 2 ** 31 else 4
    return n_elems * k * 4 + n_vertices * cfg["dim"] * 8 + nnz * 12 + (n_rows + 1) * w_rp + n_rows * 8


class ClockSampler:
    """Samples SM clock + throttle reasons through NVML during the timed region."""

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv, self.h = nv, nv.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        except Exception as e:  # no NVML: report why
            self.nv, self.err = None, str(e)
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        names = {}
        if self.nv:
            nv = self.nv
            for attr, name in [("nvmlClocksEventReasonHwSlowdown", "hw_slowdown"),
                               ("nvmlClocksEventReasonHwThermalSlowdown", "hw_thermal_slowdown"),
                               ("nvmlClocksEventReasonSwThermalSlowdown", "sw_thermal_slowdown"),
                               ("nvmlClocksEventReasonSwPowerCap", "sw_power_cap"),
                               ("nvmlClocksEventReasonHwPowerBrakeSlowdown", "hw_power_brake_slowdown")]:
                if hasattr(nv, attr):
                    names[getattr(nv, attr)] = name
        while not self._stop.is_set():
            if self.nv:
                try:
                    self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                    r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                    for bit, name in names.items():
                        if r & bit:
                            self.reasons.add(name)
                except Exception:
                    pass
            time.sleep(0.002)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join()

    def summary(self):
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# --------------------------------------------------------------------------
# reference CPU arm

def host_info():
    """always print nproc, the lscpu model, OMP_NUM_THREADS,
    the compiler and flags with a CPU number."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    info = {"nproc": os.cpu_count(), "cpu_model": model, "omp_num_threads": os.environ.get("OMP_NUM_THREADS")}
    try:
        import pyoracle as po
        if po.ref_available():
            info["reference_build"] = po.ref().ffref_build_info().decode()
    except Exception:
        pass
    return info


def cpu_reference_sample(cfg, target_s=2.0):
    """Reference CPU assembly on the box's host cores, ON THE CONFIGURED MESH.

    oracle/_ref is the unmodified reference library (symbolic CAS + IR VM +
    binary-search scatter + OpenMP atomics, all host threads):
      2D P1 (C1): the reference pipeline unchanged -- build_sparsity, then
        assemble_sparse(CompiledEvaluator) in parallel mode over the whole
        512^2 mesh every step (criterion 9, acceptance.cpp:292-327).
      3D scalar (C2/C3/C4/NS): the reference's CAS + IR VM through the 3D
        restatement of instantiate/run_assembly_block (oracle/ref_harness.cpp)
        over the full mesh and its full CSR (built once, outside the timer,
        acceptance.cpp:295-296); each step is a bounded, strided sample of the
        mesh's elements (every stride-th element, so the sample touches the
        whole CSR like the full pass), sized to ~target_s.
      Vector P2 (C5): no reference implementation; the C restatement on a
        Kuhn 8^3 sample (same element type and form; not the same mesh).
    Returns step() -> (elements, seconds), kind, workers, desc, same_mesh,
    (elements, dofs, nnz) of the configured workload."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po

    workers = os.cpu_count() or 1
    if cfg.get("ncomp", 1) > 1:
        n_s = 8
        coords, vconn = po.kuhn_mesh(n_s)
        dconn, nd = po.p2_dofs_kuhn(n_s, vconn)
        rp, ci = po.build_pattern(dconn, nd)
        vrp, vci = po.block_pattern(rp, ci, cfg["ncomp"])
        E = vconn.shape[0]

        def step():
            t = time.perf_counter()
            po.assemble_elasticity(cfg["dim"], cfg["degree"], cfg["quad"], coords, vconn, dconn, vrp, vci)
            return E, time.perf_counter() - t
        desc = (f"C restatement (oracle/femoracle.c, 1 thread): all {E} elements of a Kuhn {n_s}^3 vector P2 mesh "
                f"(the reference has no vector forms; not the {cfg['n']}^3 mesh)")
        n = cfg["n"]
        nnz_node = 230 * n ** 3 + 138 * n ** 2 + 24 * n + 1   # SURVEY Appendix A (Kuhn P2)
        sizes = (6 * n ** 3, (2 * n + 1) ** 3, cfg["ncomp"] ** 2 * nnz_node)
        return step, "port", 1, desc, False, sizes
    if not po.ref_available():
        raise RuntimeError("oracle/_ref (the reference library) is not built")
    n = cfg["n"]
    if cfg["dim"] == 2:
        if cfg["degree"] != 1:
            raise RuntimeError("the reference implements 2D P1 only")
        coords, vconn = po.unit_square_mesh(n)
        h = po.RefHarness(2, 1, coords, vconn, vconn, coords.shape[0], cfg["form"], cfg["quad"])
        E = vconn.shape[0]

        def step():
            t = time.perf_counter()
            h.assemble(workers=workers)
            return E, time.perf_counter() - t
        desc = (f"reference library (oracle/_ref): assemble_sparse(CompiledEvaluator), parallel mode, {workers} "
                f"workers, the whole {n}^2 mesh ({E} elements) per step; build_sparsity outside the timer")
        return step, "reference", workers, desc, True, (E, coords.shape[0], h.nnz)
    coords, vconn = po.kuhn_mesh(n)
    dconn, nd = (vconn, coords.shape[0]) if cfg["degree"] == 1 else po.p2_dofs_kuhn(n, vconn)
    t = time.perf_counter()
    rp, ci = po.build_pattern(dconn, nd)
    pattern_s = time.perf_counter() - t
    h = po.RefHarness(3, cfg["degree"], coords, vconn, dconn, nd, cfg["form"], cfg["quad"], pattern=(rp, ci))
    E = vconn.shape[0]
    values = np.zeros(h.nnz)
    rhs = np.zeros(nd)
    values[:] = 0.0   # touch every page outside the timer
    rhs[:] = 0.0
    probe = min(E, 4 * workers * 64)
    h.assemble_sample(values, rhs, workers, 0, max(E // probe, 1), probe)   # warm (thread scratch, caches)
    t = time.perf_counter()
    h.assemble_sample(values, rhs, workers, 1 % max(E // probe, 1), max(E // probe, 1), probe)
    rate = probe / max(time.perf_counter() - t, 1e-6)
    count = int(min(E, max(probe, rate * target_s)))
    stride = max(E // count, 1)
    state = {"i": 0}

    def step():
        first = state["i"] % stride
        state["i"] += 1
        t = time.perf_counter()
        h.assemble_sample(values, rhs, workers, first, stride, count)
        return count, time.perf_counter() - t
    desc = (f"reference library (oracle/_ref: CAS + IR VM + binary-search scatter + atomic adds, "
            f"{workers} OpenMP threads) on the full Kuhn {n}^3 mesh and its full CSR ({h.nnz} nnz, built in "
            f"{pattern_s:.1f} s outside the timer): per step every {stride}-th element ({count} of {E})")
    return step, "reference", workers, desc, True, (E, nd, h.nnz)


def run_reference_arm(args, cfg, rank, world):
    if rank != 0:
        return
    step, kind, workers, desc, same, sizes = cpu_reference_sample(cfg, target_s=args.ref_step_s)
    for _ in range(args.warmup):
        step()
    elems, secs = 0, 0.0
    for _ in range(args.steps):
        e, s = step()
        elems += e
        secs += s
    value = elems / secs
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (deterministic structured mesh)",
            "config": workload_config(cfg, world, *sizes),
            "sample": desc, "same_mesh": same,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": kind, "sample": desc,
                             "same_mesh": same, "host": host_info()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
# our arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="ns", choices=sorted(CONFIGS))
    ap.add_argument("--size", "--n", dest="n", type=int, default=0, help="override mesh resolution")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-step-s", type=float, default=2.0)
    ap.add_argument("--block", type=int, default=0, help="element-kernel CTA size (0: by body, 32 pointwise / 128)")
    ap.add_argument("--strategy", default="auto")
    ap.add_argument("--scatter", default="auto", choices=["auto", "gather", "atomic"],
                    help="auto: both scatters timed on this config before the run, the faster one kept")
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="N>1: strong (default, SURVEY §8e) = contiguous DOF row blocks of the one configured "
                         "mesh, halo elements duplicated; weak = the 1-GPU workload stacked N times")
    ap.add_argument("--emulate-rank", default="", help="R/N: time rank R's row block of an N-rank run on one GPU")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.n:
        cfg["n"] = args.n
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        return run_reference_arm(args, cfg, rank, world)

    import torch
    import torch.distributed as dist

    # FF_BENCH_SHARE_GPU=1 (testing only): several ranks on one GPU over gloo,
    # to exercise the multi-rank path where only one device is available
    share = os.environ.get("FF_BENCH_SHARE_GPU") == "1"
    if share:
        local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1802_03433_b200 import femforge as ff
    from paper_1802_03433_b200 import rowblocks

    weak = world > 1 and args.scaling == "weak"
    if weak:
        # weak scaling: the single-GPU cell stacked `world` times along the last
        # axis; each rank builds only its slab (own cell + one halo layer)
        coords, vconn_l, dconn_l, n_dofs, rb, re, E = rowblocks.weak_slab(ff, cfg["dim"], cfg["degree"], cfg["n"],
                                                                          world, rank)
        if dconn_l is None:
            dconn_l = vconn_l
        vconn = vconn_l
    else:
        coords, vconn, dconn, n_dofs = make_mesh(ff, cfg)
        E = vconn.shape[0]
        # --emulate-rank R/N (single GPU, diagnostics only): rank R's row block of
        # an N-rank strong-scaling run, to predict the per-rank step time
        emu = tuple(int(v) for v in args.emulate_rank.split("/")) if args.emulate_rank else None
        rb, re = rowblocks.row_block(n_dofs, emu[1], emu[0]) if emu else rowblocks.row_block(n_dofs, world, rank)
        if world > 1 or emu:  # strong scaling: row blocks of the one mesh
            ids = rowblocks.local_elements(dconn, rb, re)   # owned + halo elements
            vconn_l, dconn_l = np.ascontiguousarray(vconn[ids]), np.ascontiguousarray(dconn[ids])
        else:
            vconn_l, dconn_l = vconn, dconn
    ctx = ff.Context(local)
    ctx.set_scatter(args.scatter)
    ncomp = cfg.get("ncomp", 1)
    t = time.perf_counter()
    if ncomp > 1:   # vector P2 elasticity: 3x3 blocks of scalar forms
        bb, bl = ff.elasticity_text(cfg["dim"])
        form = ff.Form.blocked(ctx, cfg["dim"], cfg["degree"], ncomp, bb, bl, quad_rule=cfg["quad"],
                               strategy=args.strategy)
    else:
        bil, lin = ff.named_form(cfg["form"], cfg["dim"])
        form = ff.Form(ctx, cfg["dim"], cfg["degree"], bil, lin, quad_rule=cfg["quad"], strategy=args.strategy,
                       block_size=args.block)
    compile_ms = 1e3 * (time.perf_counter() - t)
    mesh = ff.Mesh(ctx, cfg["dim"], coords, vconn_l, None if cfg["degree"] == 1 else dconn_l, n_dofs, ncomp=ncomp)
    t = time.perf_counter()
    pat = ff.Pattern(ctx, mesh, ncomp * rb, ncomp * re)
    pattern_ms = 1e3 * (time.perf_counter() - t)
    t = time.perf_counter()
    pat.prepare(mesh)
    plan_ms = 1e3 * (time.perf_counter() - t)
    values = torch.empty(pat.nnz, dtype=torch.float64, device="cuda")
    rhs = torch.empty(pat.n_rows, dtype=torch.float64, device="cuda")
    stream = torch.cuda.Stream()       # every launch and every event on this one stream
    sp = stream.cuda_stream
    calibration = None
    if args.scatter == "auto":         # north star (3): the scatter chosen from measured times on this config
        calibration = pat.calibrate_scatter(form, mesh, values.data_ptr(), rhs.data_ptr(), sp)
    scatter = pat.scatter_for(form)   # what actually runs (gather falls back to atomic for pointwise forms)
    gather_info = pat.gather_info(mesh) if scatter == "gather" else None
    l2_bytes = 126 * 2 ** 20
    need_flush = values.numel() * 8 < 2 * l2_bytes
    flush = torch.empty(2 * l2_bytes // 4, dtype=torch.int32, device="cuda") if need_flush else None

    def step():
        ff.assemble_device(form, mesh, pat, values.data_ptr(), rhs.data_ptr(), sp)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ctx.check()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        for i in range(args.steps):
            if flush is not None:
                with torch.cuda.stream(stream):
                    flush.fill_(i)
            ev[i][0].record(stream)
            if scatter == "atomic":  # K0 and K2 timed separately
                ff.assemble_device_ex(form, mesh, pat, values.data_ptr(), rhs.data_ptr(), sp, ff.FF_ZERO_ONLY)
                ev[i][1].record(stream)
                ff.assemble_device_ex(form, mesh, pat, values.data_ptr(), rhs.data_ptr(), sp, ff.FF_SKIP_ZERO)
            else:  # atomic-free scatters write every value once: no K0. The whole
                # step is one ff_assemble_device call (a replayed CUDA graph of
                # K2a + class + generic row kernels for the gather)
                ev[i][1].record(stream)
                step()
            ev[i][2].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ctx.check()  # device-side errors (degenerate element / missing column) fail the run
    step_ms = float(np.mean([a.elapsed_time(c) for a, b, c in ev]))
    k0_ms = float(np.mean([a.elapsed_time(b) for a, b, c in ev]))
    k2_ms = float(np.mean([b.elapsed_time(c) for a, b, c in ev]))
    if scatter == "gather":  # phase split (diagnostic, separate untimed-for-value run)
        evp = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
        for i in range(args.steps):
            if flush is not None:
                with torch.cuda.stream(stream):
                    flush.fill_(i)
            evp[i][0].record(stream)
            ff.assemble_device_ex(form, mesh, pat, values.data_ptr(), rhs.data_ptr(), sp, ff.FF_GATHER_INVARIANTS_ONLY)
            evp[i][1].record(stream)
            ff.assemble_device_ex(form, mesh, pat, values.data_ptr(), rhs.data_ptr(), sp, ff.FF_GATHER_ROWS_ONLY)
            evp[i][2].record(stream)
        torch.cuda.synchronize()
        k0_ms = float(np.mean([a.elapsed_time(b) for a, b, c in evp]))
        k2_ms = float(np.mean([b.elapsed_time(c) for a, b, c in evp]))
    times = torch.tensor([step_ms, k0_ms, k2_ms], dtype=torch.float64, device="cpu" if share else "cuda")
    if world > 1:
        dist.all_reduce(times, op=dist.ReduceOp.MAX)
    step_ms, k0_ms, k2_ms = times.tolist()

    # end to end through the public API: pinned host inputs -> H2D, pattern
    # re-validation, K0 + K2, D2H of values and rhs, every step
    e2e = None
    e2e_note = None
    if args.e2e_steps > 0 and pat.nnz * 8 * 2 > 120e9:   # pinned host + device copies of the values
        e2e_note = f"e2e skipped: {pat.nnz * 8 / 1e9:.0f} GB of values per copy (run with --gpus 8: 1/8 per rank)"
    elif args.e2e_steps > 0:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
        hc, hv = pin(coords), pin(vconn_l)
        hd = pin(dconn_l) if cfg["degree"] > 1 else None
        hval = torch.empty(pat.nnz, dtype=torch.float64).pin_memory().numpy()
        hrhs = torch.empty(pat.n_rows, dtype=torch.float64).pin_memory().numpy()
        ff.assemble(form, mesh, pat, hc, hv, hd, hval, hrhs)  # warm
        if world > 1:
            dist.barrier()
        t = time.perf_counter()
        for _ in range(args.e2e_steps):
            ff.assemble(form, mesh, pat, hc, hv, hd, hval, hrhs)
        e2e_s = torch.tensor([(time.perf_counter() - t) / args.e2e_steps], dtype=torch.float64,
                             device="cpu" if share else "cuda")
        if world > 1:
            dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
        h2d = hc.nbytes + hv.nbytes + (hd.nbytes if hd is not None else 0)
        e2e = {"value": E / float(e2e_s), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(hval.nbytes + hrhs.nbytes), "ms_per_step": 1e3 * float(e2e_s)}

    nnz_tot = pat.nnz
    dofs_tot = n_dofs
    if world > 1:  # global CSR offsets: exclusive prefix over the ranks' (rows, nnz), SURVEY §8e
        _, _, rows_tot, nnz_tot = rowblocks.global_offsets(pat.nnz, pat.n_rows)
        dofs_tot = rows_tot // ncomp
    if rank != 0:
        dist.destroy_process_group()
        return
    peak, peak_src = measured_peaks()
    B = algorithmic_bytes(cfg, vconn_l.shape[0], coords.shape[0], pat.n_rows, pat.nnz)
    F = model_flops(cfg) * vconn_l.shape[0]   # SURVEY.md §8d flop model
    # the dominant kernel(s): the whole atomic-free step (K2a + K2b) for the
    # gather, K2 for the atomic scatter (K0 is a separate memset-like kernel)
    kern_ms = step_ms if scatter == "gather" else k2_ms
    achieved = B / (kern_ms * 1e-3) / 1e9
    info = form.info
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"traffic_{args.config}_n{cfg['n']}_{scatter}.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            stepf, kind, workers, desc, same, _ = cpu_reference_sample(cfg)
            e, s = stepf()
            cpu = {"value": e / s, "unit": UNIT, "cores": workers, "kind": kind, "sample": desc,
                   "same_mesh": same, "host": host_info()}
        except Exception as ex:  # never let the baseline hide the GPU number
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port", "sample": f"failed: {ex}"}
    value = E / (step_ms * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": "weak" if weak else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (deterministic structured mesh)",
        "config": workload_config(cfg, world, E, dofs_tot, nnz_tot, weak),
        "detail": {"step": STEP_DESC[scatter] + ", inputs resident in HBM", "scatter": scatter,
                   "k0_ms": k0_ms if scatter == "atomic" else 0.0,
                   "k2a_ms": k0_ms if scatter == "gather" else None,
                   "k2_ms": k2_ms, "pattern_build_ms": pattern_ms, "slot_plan_ms": plan_ms,
                   "scatter_calibration": calibration,
                   "gather_plan": gather_info,
                   "nvrtc_compile_ms": compile_ms, "strategy": info["strategy"], "registers": info["registers"],
                   "flops_per_element": info["flops_per_element"],
                   "hbm_gbs_step": B / (step_ms * 1e-3) / 1e9},
        # the binding roofline, and (C3/NS sit at the ridge) the
        # other fraction beside it; flops = the SURVEY §8d model
        "roofline": ({"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                      "fp64": {"achieved_tflops": F / (kern_ms * 1e-3) / 1e12, "peak_tflops": FP64_PEAK_TFLOPS,
                               "frac": F / (kern_ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
                               "flops_per_element_model": model_flops(cfg), "peak_source": FP64_PEAK_SOURCE}}
                     if info["flops_per_element"] * vconn_l.shape[0] / B <= FP64_PEAK_TFLOPS * 1e3 / peak else
                     {"bound": "fp64", "achieved": F / (kern_ms * 1e-3) / 1e12, "peak": FP64_PEAK_TFLOPS,
                      "unit": "TFLOP/s", "frac": F / (kern_ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
                      "peak_note": FP64_PEAK_SOURCE + "; flops = SURVEY.md §8d model",
                      "flops_per_element_model": model_flops(cfg),
                      "hbm": {"achieved_gbs": achieved, "peak_gbs": peak, "frac": achieved / peak}}) | {
                     "traffic": traffic,
                     "kernel": KERNEL_DESC[scatter],
                     "bytes_per_launch": int(B), "peak_source": peak_src},
        "cpu_baseline": cpu,
        "e2e": e2e if e2e is not None else ({"skipped": e2e_note} if e2e_note else None),
        # ours only (the L2 flush is a torch fill): gather = K2a + class + generic
        # launches (plan-dependent), atomic = K0 + K2
        "gpu_launches": (gather_info["launches"] if scatter == "gather" else 2)
                        * args.steps,
        "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
