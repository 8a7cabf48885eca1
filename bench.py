#!/usr/bin/env python
"""Benchmark: gate applications/s on the BASELINE.json hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N=1 workload = BASELINE.json configs[1]: random layer circuit, n=26
complex128, 200 layers x (26 one-qubit gates + 13 CNOTs) = 7,800 gate
applications per step, from |0...0>, on one B200.  A step resets the 1 GiB
state (> 126 MB L2, so no L2 flush is needed) and applies the whole circuit.

N>1 (torchrun, one process per GPU): weak scaling over the partitioned
engine -- n = 26 + log2(N) qubits, k = log2(N) global qubits, so every GPU
holds a 2^26-amplitude slab and CNOTs touching a global qubit exchange with
the partner rank (paper_1801_01037_b200.dist).

Extra keys on the one JSON line:
  roofline      dominant kernel's algorithmic bytes / its CUDA-event time
                (libsvb's in-library event profiler, on the launch stream,
                over the timed region) vs MEASURED_PEAKS.json hbm_gbs;
  cpu_baseline  the reference's own compiled kernel (oracle/_ref, built
                from /root/reference by build()) on all host cores, over a
                bounded prefix of the same circuit;
  e2e           same metric through the public host-memory batch call
                device.simulate_batch (pinned H2D + run + D2H per step,
                neighbouring steps overlapped; `serial`: one call per step);
  local_gate_sweep  BASELINE configs[2]: n=30, one Haar U per target
                t=0..29 x 10 reps, per-target HBM GB/s (one launch per
                application, no fusion);
  clocks        nvidia-smi samples during the timed region.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

N_QUBITS = 26
LAYERS = 200
SWEEP_N = 30
SWEEP_REPS = 10
METRIC = "gate applications/s"
UNIT = "gate_apps/s"


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def peaks() -> tuple[float, str]:
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ("sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU reference (oracle/ is the checker and the CPU baseline; never the product)


def workload_config(n: int = N_QUBITS, layers: int = LAYERS) -> dict:
    """The workload keys both arms print (the driver compares the dicts);
    implementation details go in each arm's `impl` key."""
    return {"workload": f"random layer circuit n={n}, {layers} layers x ({n} 1q + {n // 2} CNOT) "
                        f"= {layers * (n + n // 2)} ops (BASELINE configs[1])",
            "n_qubits": n, "layers": layers, "ops_per_circuit": layers * (n + n // 2),
            "initial_state": "|0...0>", "state_bytes": 16 << n,
            "l2": "state 1 GiB > 126 MB L2; no flush needed"}


class CpuReference:
    """The reference's compiled stride kernel (oracle/_ref: svsim's own
    _stride_cy built from /root/reference; else the C port) applying a
    circuit op by op on host memory -- the paper's CPU path
    (kernel/__init__.py:107-134 -> _stride_cy.pyx:24-90)."""

    MODES = {"sequential": 0, "parallel_collapsed": 3}

    def __init__(self, n: int, cores: int):
        sys.path.insert(0, os.path.join(REPO, "oracle"))
        import oracle

        self.oracle = oracle
        self.ref = oracle.ref_module()
        self.kind = "reference" if self.ref is not None else "port"
        self.cores = cores
        self.amps = np.zeros(1 << n, np.complex128)
        self.reset()

    def reset(self) -> None:
        self.amps[:] = 0
        self.amps[0] = 1.0

    def apply(self, op, mode: str = "parallel_collapsed") -> None:
        g, a = op.gate, self.amps
        workers = 1 if mode == "sequential" else self.cores
        if self.ref is not None:
            m = self.MODES[mode]
            if op.control is None:
                self.ref.apply_single(a, g.q11, g.q12, g.q21, g.q22, op.target, m, workers)
            else:
                self.ref.apply_controlled(a, g.q11, g.q12, g.q21, g.q22, op.control, op.target, m, workers)
        elif op.control is None:
            self.oracle.apply_single(a, g, op.target, workers)
        else:
            self.oracle.apply_controlled(a, g, op.control, op.target, workers)

    def label(self, mode: str) -> str:
        src = "svsim _stride_cy (oracle/_ref)" if self.ref is not None else "oracle C port"
        threads = 1 if mode == "sequential" else self.cores
        return f"{src} mode {mode} x{threads}"


def cpu_reference_rate(circuit, budget_s: float, cores: int, mode: str = "parallel_collapsed") -> dict:
    """Bounded sample: the first ops of `circuit` from |0...0> for about
    budget_s seconds (the GPU arm's cpu_baseline; `sequential` is the
    paper's own mode)."""
    cpu = CpuReference(circuit.n, cores)
    done = 0
    t0 = time.perf_counter()
    for op in circuit.ops:
        cpu.apply(op, mode)
        done += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    dt = time.perf_counter() - t0
    return {"value": done / dt, "unit": UNIT, "cores": 1 if mode == "sequential" else cores, "kind": cpu.kind,
            "sample": f"first {done} of {len(circuit.ops)} ops of the n={circuit.n} random layer circuit "
                      f"(configs[1]) from |0...0>, {cpu.label(mode)}, {dt:.1f} s"}


def run_reference_arm(args) -> None:
    """--impl reference: the reference's CPU path on the whole configs[1]
    circuit.  The circuit's 7,800 ops are split into K contiguous slices;
    timed step i applies slice i, so the K timed steps apply the complete
    circuit once, from |0...0>, on every host core (mode parallel_collapsed,
    the reference's fastest).  Warm-up steps apply the first W slices to a
    scratch run that is then reset.  value = 7,800 ops / total timed time.
    Also a bounded sample of the paper's own `sequential` mode."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1801_01037_b200 import workloads

    n = N_QUBITS
    circuit = workloads.random_layer_circuit(n, LAYERS)
    ops = circuit.ops
    cores = host_cores()
    steps, warm = max(args.steps, 1), max(args.warmup, 0)
    bounds = [len(ops) * i // steps for i in range(steps + 1)]
    cpu = CpuReference(n, cores)
    t0 = time.perf_counter()
    for i in range(warm):
        for op in ops[bounds[i % steps]:bounds[i % steps + 1]]:
            cpu.apply(op)
    warm_s = time.perf_counter() - t0
    cpu.reset()
    per_step = []
    for i in range(steps):
        t0 = time.perf_counter()
        for op in ops[bounds[i]:bounds[i + 1]]:
            cpu.apply(op)
        per_step.append(time.perf_counter() - t0)
    total = sum(per_step)
    norm = float(np.vdot(cpu.amps, cpu.amps).real)
    value = len(ops) / total
    seq = None if args.no_sequential else cpu_reference_rate(circuit, args.seq_budget, cores, "sequential")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": steps, "warmup": warm,
        "ms_per_step": 1e3 * total / steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "c128", "data": "synthetic (seeded numpy PCG64 circuit, |0...0> start)",
        "config": workload_config(n, LAYERS),
        "impl_detail": {"engine": cpu.label("parallel_collapsed"),
                        "step": f"1/{steps} of the circuit: timed step i applies ops "
                                f"[{len(ops)}*i/{steps}, {len(ops)}*(i+1)/{steps}); the {steps} timed steps "
                                f"apply all {len(ops)} ops once, from |0...0>",
                        "ops_per_step": len(ops) / steps, "timed_s": round(total, 3),
                        "warmup_s": round(warm_s, 3), "norm_after_circuit": norm},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": cpu.kind,
                         "sample": f"the whole {len(ops)}-op circuit from |0...0> over the {steps} timed "
                                   f"steps, {cpu.label('parallel_collapsed')}, {total:.1f} s"},
        "sequential": seq,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm


def local_gate_sweep(n: int, reps: int, peak: float) -> dict:
    """configs[2]: per-target HBM GB/s of single general-U applications."""
    import torch

    from paper_1801_01037_b200 import _lib, device, workloads

    lib = _lib.load()
    st = device.DeviceState.random(n, seed=workloads.SEED_STATE)
    circ = workloads.sweep_ops(n, reps)
    stream = torch.cuda.current_stream()
    sp = device._stream_ptr()
    bytes_per_app = 32 * (1 << n)
    per_t = []
    for t in range(n):
        q = _lib.gate_array(circ.ops[t * reps].gate)
        # repetition 1 warms the launch path untimed; 2..reps are timed, so the
        # final state is exactly the 300 configs[2] applications
        # (tests/test_gpu_large.py compares it with the oracle)
        _lib.check(lib.svb_apply_1q(st.ptr, 1 << n, q, t, sp))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps - 1):
            _lib.check(lib.svb_apply_1q(st.ptr, 1 << n, q, t, sp))
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / (reps - 1)
        per_t.append(bytes_per_app / ms / 1e6)
    nrm = device.norm2(st)
    del st
    torch.cuda.empty_cache()
    arr = np.array(per_t)
    return {"config": f"n={n}, Haar U on t=0..{n - 1} x {reps} reps (configs[2])",
            "gbs_min": round(float(arr.min()), 1), "gbs_median": round(float(np.median(arr)), 1),
            "gbs_max": round(float(arr.max()), 1),
            "frac_min": round(float(arr.min()) / peak, 4), "frac_median": round(float(np.median(arr)) / peak, 4),
            "apps_per_s_median": round(float(np.median(arr)) * 1e9 / bytes_per_app, 1),
            "per_target_gbs": [round(float(x), 1) for x in arr],
            "norm_after": nrm, "bytes_per_app": bytes_per_app}


def qft20_rate(args, reps: int = 20) -> dict:
    """BASELINE configs[0] on the GPU: QFT n=20 on the seeded Gaussian state
    (16 MiB, L2-resident), device-resident, the bench's arithmetic mode."""
    import torch

    from paper_1801_01037_b200 import device, workloads

    n = 20
    circ = workloads.qft_circuit(n)
    a = torch.from_numpy(workloads.seeded_state(n, workloads.SEED_STATE)).cuda()
    st = device.DeviceState(n, a.clone())
    kw = dict(fuse=not args.no_fuse, fma=args.fma, jit=args.jit)
    device.run_ops(st, circ, **kw)  # plan + compile
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        st.amps.copy_(a)
        device.run_ops(st, circ, **kw)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return {"config": "QFT n=20 on the seeded Gaussian state (configs[0]), state reset + circuit per rep",
            "ops": len(circ.ops), "ms_per_circuit": round(ms, 4),
            "gate_apps_per_s": round(len(circ.ops) / (ms / 1e3), 1),
            "passes": device.plan_passes(n, circ, fuse=not args.no_fuse, jit=args.jit)}


_COLD_CHILD = r"""
import sys, time, numpy as np
sys.path.insert(0, {repo!r})
import torch
from paper_1801_01037_b200 import _lib, device, workloads
torch.zeros(1, device="cuda")  # context up before the clock starts
circ = workloads.random_layer_circuit({n}, {layers})
a = np.zeros(1 << {n}, np.complex128); a[0] = 1
t0 = time.perf_counter()
device.simulate(circ, a, fma=True, jit=True)
print(time.perf_counter() - t0, *_lib.jit_counters())
"""


def cold_start(circuit, layers: int) -> dict:
    """First call of a circuit the process has never seen, through the public
    host API (device.simulate: H2D + run + D2H of the 1 GiB state):
    * jit="async": interpreter run now, specialised passes compiled in the
      background (on-disk cubin cache empty: a fresh per-run directory);
    * a NEW process with the cubins now on disk (jit=True, nothing compiled);
    * for comparison the synchronous jit=True first step is first_step_s."""
    from paper_1801_01037_b200 import _lib, device

    n = circuit.n
    a = np.zeros(1 << n, np.complex128)
    a[0] = 1.0
    t0 = time.perf_counter()
    device.simulate(circuit, a, fma=True, jit="async")
    first = time.perf_counter() - t0
    _lib.jit_wait()
    ready = time.perf_counter() - t0
    hits, comps = _lib.jit_counters()
    out = {"first_call_s": round(first, 3), "first_call_gate_apps_per_s": round(len(circuit.ops) / first, 1),
           "first_call_path": "interpreter (quick plan) while NVRTC compiles in the background",
           "background_compile_done_s": round(ready, 3), "cubins_compiled": comps, "cubins_from_disk": hits}
    r = subprocess.run([sys.executable, "-c", _COLD_CHILD.format(repo=REPO, n=n, layers=layers)],
                       capture_output=True, text=True, timeout=900)
    if r.returncode == 0:
        t, h, c = r.stdout.split()[-3:]
        out["new_process_first_call_s"] = round(float(t), 3)
        out["new_process_cubins"] = {"from_disk": int(h), "compiled": int(c)}
    else:
        out["new_process_error"] = r.stderr[-300:]
    return out


def seam_rates(circuit) -> dict:
    """Gate applications/s through the reference-facing seams on HOST arrays:
    * backend.apply_single / apply_controlled -- svsim's kernel-backend
      contract (kernel/__init__.py:107-134), one gate per synchronous call,
      the whole state through PCIe each call (streamed in 64 MiB units);
      configs[1]'s circuit at n=20 and its first two layers at n=26;
    * engine.run_circuit(..., fused="fast") at k=0 -- the reference engine's
      entry point (engine.py:457-512) with the local ops fused, GateStats per
      gate, gather() to the host included: configs[1] whole."""
    from paper_1801_01037_b200 import backend, engine, workloads
    from paper_1801_01037_b200.partition import PartitionPlan

    out = {}
    for n, layers, nops in ((20, 10, None), (26, 200, 78)):
        circ = workloads.random_layer_circuit(n, layers) if n != circuit.n else circuit
        ops = circ.ops[:nops] if nops else circ.ops
        a = np.zeros(1 << n, np.complex128)
        a[0] = 1.0

        def apply(op):
            g = op.gate
            if op.control is None:
                backend.apply_single(a, g.q11, g.q12, g.q21, g.q22, op.target, 3, 1)
            else:
                backend.apply_controlled(a, g.q11, g.q12, g.q21, g.q22, op.control, op.target, 3, 1)

        apply(ops[0])  # warm: staging buffers, page-locking of `a`
        t0 = time.perf_counter()
        for op in ops:
            apply(op)
        dt = time.perf_counter() - t0
        out[f"backend_n{n}"] = {"value": round(len(ops) / dt, 1), "unit": UNIT, "ops": len(ops),
                                "bytes_per_call": 2 * (16 << n)}
    t0 = time.perf_counter()
    ds, stats = engine.run_circuit(circuit, PartitionPlan(circuit.n, 0), fused="fast")
    t1 = time.perf_counter()
    amps = engine.gather(ds).amps
    dt = time.perf_counter() - t0
    ds.close()
    out["engine_fused_n%d" % circuit.n] = {"value": round(len(circuit.ops) / dt, 1), "unit": UNIT,
                                           "run_circuit_s": round(t1 - t0, 3), "gather_s": round(dt - (t1 - t0), 3),
                                           "gate_stats": len(stats), "norm": float(np.vdot(amps, amps).real),
                                           "api": "engine.run_circuit(..., fused='fast') + gather() to a new "
                                                  "host array, plan and kernels already cached"}
    return out


def qft33_rate(args, reps: int = 3) -> dict:
    """BASELINE configs[3]'s workload on ONE GPU -- QFT n=33 (128 GiB state)
    from the seeded device-drawn Gaussian state, the bench's arithmetic mode,
    one QFT per repetition over the current state: the N=1 point of the
    configs[3] strong-scaling curve that `bench.py --gpus N` (N=2/4/8) prints
    as its headline.  Known answers are tested in tests/test_gpu_large.py."""
    import torch

    from paper_1801_01037_b200 import device, workloads

    n = 33
    circ = workloads.qft_circuit(n)
    torch.cuda.empty_cache()
    st = device.DeviceState.random(n, seed=7)
    kw = dict(fuse=not args.no_fuse, fma=args.fma, jit=args.jit)
    device.run_ops(st, circ, **kw)  # plan + compile
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        device.run_ops(st, circ, **kw)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    nrm = device.norm2(st)
    del st
    torch.cuda.empty_cache()
    return {"config": "QFT n=33 on one GPU (BASELINE configs[3] workload, N=1 point of its strong scaling)",
            "ops": len(circ.ops), "ms_per_circuit": round(ms, 3),
            "gate_apps_per_s": round(len(circ.ops) / (ms / 1e3), 1),
            "hbm_passes": device.plan_passes(n, circ, fuse=not args.no_fuse, jit=args.jit),
            "state_bytes": 16 << n, "norm_after": nrm}


def run_gpu_arm(args) -> None:
    import tempfile

    # a fresh on-disk JIT cache per run: the cold-start numbers never ride on
    # a cache an earlier run left behind (the child process inherits it)
    os.environ.setdefault("SVB_JIT_CACHE", tempfile.mkdtemp(prefix="svb-jit-"))
    import torch

    from paper_1801_01037_b200 import _lib, device, workloads

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or os.environ.get("SVB_BENCH_DIST") == "1":  # (=1: the N>1 engine at world 1, a smoke test)
        from paper_1801_01037_b200 import dist

        dist.bench_main(args, clock_cls=ClockSampler, peaks_fn=peaks)
        return

    lib = _lib.load()
    torch.cuda.set_device(0)
    n = N_QUBITS
    circuit = workloads.random_layer_circuit(n, LAYERS)
    nops = len(circuit.ops)
    ops_arr, _ = _lib.ops_array(circuit.ops)
    flags = _lib.run_flags(fuse=not args.no_fuse, fma=args.fma, jit=args.jit)
    passes = device.plan_passes(n, circuit, fuse=not args.no_fuse, jit=args.jit)
    cold = None if (args.no_cold or not args.jit) else cold_start(circuit, LAYERS)
    st = device.DeviceState.zeros(n)
    stream = torch.cuda.current_stream()
    sp = device._stream_ptr()

    def step():
        st.amps.zero_()
        st.amps[0] = 1.0
        _lib.check(lib.svb_run_ops(st.ptr, 1 << n, ops_arr, nops, flags, sp), "run_ops")

    # first warm-up step plans the circuit and (with JIT) compiles its passes
    t_first = time.perf_counter()
    step()
    torch.cuda.synchronize()
    first_step_s = time.perf_counter() - t_first
    for _ in range(max(args.warmup - 1, 0)):
        step()
    torch.cuda.synchronize()
    _lib.profile_enable(os.environ.get("SVB_BENCH_NOPROF") != "1")  # (=1: measure the profiler's cost)
    launches0 = _lib.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    launches = _lib.launch_count() - launches0
    prof = _lib.profile_read()
    _lib.profile_enable(False)
    norm_after = device.norm2(st)
    value = nops * args.steps / (ms / 1e3)

    peak, peak_src = peaks()
    dom = max(prof.items(), key=lambda kv: kv[1][1]) if prof else None
    roofline = None
    if dom:
        name, (cnt, tms, nbytes) = dom
        achieved = nbytes / (tms / 1e3) / 1e9
        traffic = None
        tpath = os.path.join(REPO, "profiles", "traffic.json")
        if os.path.exists(tpath):
            with open(tpath) as f:
                traffic = json.load(f).get(name)
        roofline = {"bound": "hbm", "kernel": name, "achieved": round(achieved, 1), "peak": peak,
                    "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                    "alg_bytes_per_launch": nbytes // cnt, "avg_launch_ms": round(tms / cnt, 4),
                    "launches": cnt, "share_of_step": round(tms / ms, 4), "peak_source": peak_src}
    kernels = {k: {"launches": v[0], "ms": round(v[1], 3), "gbs": round(v[2] / (v[1] / 1e3) / 1e9, 1)}
               for k, v in prof.items()}

    # e2e through the public host-memory calls, pinned buffers.  Headline:
    # simulate_batch (svb_host_run_ops_batch) over `steps` input states --
    # every step copies its 1 GiB state in and its result out, overlapped
    # with the neighbouring steps' runs; also one simulate call per step
    # (no overlap) for comparison
    pin_in = torch.zeros(1 << n, dtype=torch.complex128).pin_memory()
    pin_in[0] = 1.0
    a_in = pin_in.numpy()
    e2e_steps = max(3, 4 * args.steps)  # a serving batch of 20 states by default; the pipeline fill (first H2D) and drain (last D2H) amortised over it
    # six pinned result buffers used round robin (the library copies results
    # out in order on one stream, so a buffer is rewritten only after it was
    # filled six states earlier)
    bufs = [torch.empty(1 << n, dtype=torch.complex128).pin_memory().numpy() for _ in range(min(e2e_steps, 6))]
    outs = [bufs[k % len(bufs)] for k in range(e2e_steps)]
    kw = dict(fuse=not args.no_fuse, fma=args.fma, jit=args.jit)
    device.simulate_batch(circuit, [a_in], [outs[0]], **kw)
    for b in bufs:
        b[:] = 0
    t0 = time.perf_counter()
    device.simulate_batch(circuit, [a_in] * e2e_steps, outs, **kw)
    e2e_dt = time.perf_counter() - t0
    e2e_norm = float(np.vdot(outs[-1], outs[-1]).real)
    e2e_same = all(np.array_equal(o, bufs[0]) for o in bufs[1:])
    serial_steps = max(1, min(args.steps, 3))
    t0 = time.perf_counter()
    for k in range(serial_steps):
        device.simulate(circuit, a_in, out=outs[k], **kw)
    serial_dt = time.perf_counter() - t0

    seam = None if args.no_seam else seam_rates(circuit)
    sweep = None if args.no_sweep else local_gate_sweep(SWEEP_N, SWEEP_REPS, peak)
    qft = None if args.no_sweep else qft20_rate(args)

    del st
    torch.cuda.empty_cache()
    qft33 = None
    if not args.no_sweep:
        try:
            qft33 = qft33_rate(args)
        except Exception as exc:  # (a GPU without 128 GiB free)
            qft33 = {"skipped": str(exc)[:200]}

    cores = host_cores()
    cpu = None
    if not args.no_cpu:
        cpu = cpu_reference_rate(circuit, args.cpu_budget, cores)

    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic (seeded numpy PCG64 circuit, |0...0> start)",
        "config": workload_config(n, LAYERS),
        "impl_detail": {"engine": "libsvb svb_run_ops (include/svb.h)", "fused": not args.no_fuse,
                        "fma": args.fma, "jit": args.jit, "hbm_passes_per_step": passes,
                        "ops_per_step": nops, "parallelism": "single GPU"},
        "roofline": roofline,
        "kernels": kernels,
        "gpu_launches": launches,
        "e2e": {"value": round(nops * e2e_steps / e2e_dt, 1), "unit": UNIT,
                "h2d_bytes_per_step": 16 << n, "d2h_bytes_per_step": 16 << n,
                "api": "paper_1801_01037_b200.device.simulate_batch (svb_host_run_ops_batch): per step "
                       "H2D + run + D2H, neighbouring steps overlapped; pinned host buffers",
                "steps": e2e_steps,
                "serial": {"value": round(nops * serial_steps / serial_dt, 1), "steps": serial_steps,
                           "api": "device.simulate (svb_host_run_ops), one synchronous call per step"}},
        "e2e_seam": seam,
        "cpu_baseline": cpu,
        "local_gate_sweep": sweep,
        "qft20": qft,
        "qft33": qft33,
        "clocks": clk.summary(),
        "check": {"norm_after_step": norm_after, "e2e_norm": e2e_norm, "e2e_outputs_identical": e2e_same},
        "cold_start": cold,
        "first_step_s": round(first_step_s, 3),  # (after cold_start: plan and kernels already built)
    }
    print(json.dumps(line), flush=True)


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-fuse", action="store_true", help="one launch per gate")
    ap.add_argument("--no-fma", dest="fma", action="store_false",
                    help="exact reference arithmetic in fused passes (default: FMA contraction, "
                         "within ~1 ulp, parity-tested <= 1e-12)")
    ap.add_argument("--no-jit", dest="jit", action="store_false",
                    help="interpret fused passes (default: compile each pass once to a straight-line "
                         "kernel with NVRTC; compile cost reported under cold_start)")
    ap.add_argument("--no-sweep", action="store_true", help="skip the configs[2] n=30 sweep")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--no-cold", action="store_true", help="skip the cold-start measurement")
    ap.add_argument("--no-seam", action="store_true", help="skip the host-seam measurements")
    ap.add_argument("--cpu-budget", type=float, default=15.0, help="seconds of CPU reference work")
    ap.add_argument("--seq-budget", type=float, default=8.0,
                    help="--impl reference: seconds of the paper's sequential mode (bounded sample)")
    ap.add_argument("--no-sequential", action="store_true", help="--impl reference: skip the sequential sample")
    args = ap.parse_args(argv)
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_gpu_arm(args)


if __name__ == "__main__":
    main()
