"""bench.py — QSVM kernel entries/s at 784 qubits (BASELINE.json metric) on 1..8 B200.

Workload (BASELINE.json configs[3], the config the 1/2/4/8-GPU metric is quoted on; it fits one
GPU): MNIST-shaped synthetic data, 784 qubits, L = 2, train Gram 10000 x 10000 (49,995,000
strict-upper entries; diagonal injected) + test-versus-train cross 2000 x 10000 (20,000,000
entries).  One step = gate build + pair sweeps of the whole job; for N > 1 the tile list is
split into contiguous ranges of equal estimated cost and every rank's sweep stores its tiles
straight into rank 0's matrices over NVLink (CUDA IPC), closed by one barrier (distributed.py).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

value       whole-job entries/s, device-resident inputs, CUDA events, max over ranks
e2e         same metric through the public API with host (pinned) buffers, H2D + D2H inside
roofline    sweep kernel, executed FP64 flops / CUDA-event launch time vs B200 FP64 peak
cpu_baseline  oracle/ (the reference's contraction restated in C) on the host cores, sampled;
            plus .reference_python: the unmodified reference package (baseline/_ref) itself,
            contract_batch(workers=os.cpu_count()) on 512 sampled pairs in a CUDA-free
            subprocess, with its amplitudes compared against this run's matrices
--impl reference  the oracle CPU baseline as the reference arm (rank 0 only)
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "QSVM kernel entries/sec at 784 qubits, 1/2/4/8 B200; % of FP64 roofline"
UNIT = "entries/s"
N_QUBITS, N_TRAIN, N_TEST, LAYERS = 784, 10000, 2000, 2
WORKLOAD = {"workload": "configs[3]: MNIST-shaped synthetic, 10-class, 784 qubits, "
                        "10000 train Gram (strict upper) + 2000x10000 test-vs-train cross",
            "qubits": N_QUBITS, "layers": LAYERS, "n_train": N_TRAIN, "n_test": N_TEST,
            "convention": "probability", "angle_bandwidth": 1.0,
            "l2": "inputs larger than L2: 150 MB gate planes + 960 MB kernel output per step"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=6)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def workload_data():
    from paper_2405_02630_b200.data import config_data

    Atr, ytr, Ate, yte = config_data(4, N_TRAIN, N_TEST, "mnist", bw=1.0)
    return Atr, Ate


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ------------------------------------------------------------------------------------------
# CPU baseline (the oracle: the reference's TN contraction restated in C, all host threads)
# ------------------------------------------------------------------------------------------
def cpu_baseline_run(Atr, Ate, seconds: float, seed: int = 0):
    from oracle import oracle

    threads = host_threads()
    rng = np.random.default_rng(seed)
    A = np.concatenate([Atr, Ate])

    def sample(P):
        return sample_pairs(rng, P)

    cal = sample(max(threads * 2, 8))
    t0 = time.perf_counter()
    oracle.amplitudes(A, A, cal, LAYERS, threads)
    rate = len(cal) / (time.perf_counter() - t0)
    P = int(max(threads * 4, min(rate * seconds, 2_000_000)))
    pairs = sample(P)
    t0 = time.perf_counter()
    oracle.amplitudes(A, A, pairs, LAYERS, threads)
    dt = time.perf_counter() - t0
    return {"value": P / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{P} pairs sampled uniformly from the workload's 69,995,000 "
                      f"(seed {seed}); oracle/qk_oracle.c complex128 TN contraction, "
                      f"{threads} pthreads on {cpu_model()}",
            "seconds": dt}


def sample_pairs(rng, P):
    """P pairs uniform over the workload's pair set (Gram strict upper + cross), as row
    indices into concat(train, test)."""
    n_gram = N_TRAIN * (N_TRAIN - 1) // 2
    total = n_gram + N_TEST * N_TRAIN
    out = np.empty((P, 2), dtype=np.int64)
    for k in range(P):
        while True:
            if rng.integers(total) < n_gram:
                i, j = rng.integers(N_TRAIN, size=2)
                if i < j:
                    out[k] = (i, j)
                    break
            else:
                out[k] = (N_TRAIN + rng.integers(N_TEST), rng.integers(N_TRAIN))
                break
    return out


def reference_python_run(Atr, Ate, n_pairs: int = 512, repeats: int = 3, seed: int = 7):
    """The unmodified reference (baseline/_ref) timed on the host cores: contract_batch over
    n_pairs sampled pairs with workers=os.cpu_count(), median of `repeats`, planning timed
    separately, in a subprocess that sees no CUDA device.  Returns the record
    and (pairs, amplitudes) for a parity check."""
    import tempfile

    script = ROOT / "tools" / "ref_baseline.py"
    if not (ROOT / "baseline" / "_ref" / "tnkernel").is_dir():
        return {"unavailable": "baseline/_ref (pip install --target of the reference) absent"}, None
    pairs = sample_pairs(np.random.default_rng(seed), n_pairs)
    with tempfile.TemporaryDirectory() as td:
        a, p, o = Path(td) / "a.npy", Path(td) / "p.npy", Path(td) / "o.json"
        np.save(a, np.concatenate([Atr, Ate]))
        np.save(p, pairs)
        env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
        try:
            subprocess.run([sys.executable, str(script), str(a), str(p), str(o), str(repeats)],
                           env=env, check=True, timeout=900, capture_output=True)
            r = json.loads(o.read_text())
        except (subprocess.SubprocessError, OSError, ValueError) as exc:
            return {"unavailable": f"reference run failed: {str(exc)[:200]}"}, None
    rec = {"value": r["entries_per_s"], "unit": UNIT, "cores": r["workers"], "kind": "reference",
           "sample": f"{len(pairs)} pairs sampled uniformly from the workload (seed {seed}); "
                     "unmodified reference tnkernel.engine.contract_batch(simplified kernel "
                     f"network, plan_contraction path, workers={r['workers']}) on "
                     f"{cpu_model()}, median of {repeats}",
           "plan_s": r["plan_s"], "runs_s": r["runs_s"]}
    return rec, (pairs, np.asarray(r["amplitudes_re"]))


def parity_vs_reference(Atr, Ate, pairs, amp, K_ours):
    """The engine's K on the reference's sampled pairs against the reference's amplitudes.

    Gates: |dK| <= 1e-12 absolute on every pair (north star); the amplitude
    gate |d amp| <= 1e-9 |amp_ref| + 1e-300 on every pair whose reference value is defined
    to that relative precision by its input.  At angle bandwidth 1 most |amp| are ~1e-150 and
    below, and the pairs whose amplitude is a product of cos(pi_double / 2) = 6.1e-17 factors
    (an ink pixel x = pi * 1.0 against a background 0) move by 1e3-1e9x under a 1-ulp change of
    every angle, in the reference itself: their relative value is rounding noise of the input,
    and only the absolute gate applies to them.  The conditioning is measured with the oracle
    (the pinned restatement of the reference's contraction) at angles one ulp up and down."""
    from oracle import oracle

    A = np.concatenate([Atr, Ate])
    K_ref = amp * amp
    k_up = np.real(oracle.amplitudes(np.nextafter(A, 10.0), np.nextafter(A, 10.0), pairs,
                                     LAYERS, host_threads())) ** 2
    k_dn = np.real(oracle.amplitudes(np.nextafter(A, -10.0), np.nextafter(A, -10.0), pairs,
                                     LAYERS, host_threads())) ** 2
    spread = np.maximum(np.abs(k_up - K_ref), np.abs(k_dn - K_ref))
    normal = K_ref > 1e-300
    cond_ok = normal & (spread <= 1e-9 * K_ref)
    a_ours = np.sqrt(K_ours)
    ratio = np.abs(a_ours - np.abs(amp)) / (1e-9 * np.abs(amp) + 1e-300)
    return {"pairs": int(len(pairs)),
            "max_abs_dK": float(np.abs(K_ours - K_ref).max()), "abs_gate": 1e-12,
            "pairs_K_normal": int(normal.sum()),
            "pairs_well_conditioned": int(cond_ok.sum()),
            "amp_gate_max_ratio_well_conditioned": float(ratio[cond_ok].max())
            if cond_ok.any() else None,
            "max_rel_dK_well_conditioned": float(np.max(
                np.abs(K_ours[cond_ok] - K_ref[cond_ok]) / K_ref[cond_ok])) if cond_ok.any()
            else None,
            "ill_conditioned_note": "normal-K pairs whose reference K moves by more than 1e-9 "
                                    "relative under a 1-ulp change of the angles: "
                                    f"{int((normal & ~cond_ok).sum())}"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    Atr, Ate = workload_data()
    per_step = max(2.0, min(8.0, 120.0 / max(1, args.steps + args.warmup)))
    vals = []
    for s in range(args.warmup + args.steps):
        r = cpu_baseline_run(Atr, Ate, per_step, seed=s)
        if s >= args.warmup:
            vals.append(r)
    v = float(np.median([r["value"] for r in vals]))
    out = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.median([r["seconds"] for r in vals])),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
           "config": dict(WORKLOAD),
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": vals[0]["cores"], "kind": "port",
                            "sample": vals[0]["sample"]},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "note": "reference = oracle/ port of the reference's tensor-network contraction "
                   "(complex128 C, all host threads; the conservative arm: ~140x faster than "
                   "the Python reference itself, which is timed alongside as "
                   "reference_python); each step times a bounded pair sample of the same "
                   "workload"}
    if not args.no_cpu_baseline:
        out["reference_python"] = reference_python_run(Atr, Ate)[0]
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------------------------------
# clocks sampling (nvidia-smi during the timed region)
# ------------------------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = Path(f"/tmp/qk_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, power, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.path.read_text().splitlines()[1:]:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1].split()[0]))
                smax.append(float(f[2].split()[0]))
                power.append(float(f[3].split()[0]))
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        loaded = [s for s, p in zip(sm, power) if p > 0.5 * max(power)] if power else sm
        return {"sm_mhz": float(np.median(loaded)) if loaded else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(power) if power else None}


# ------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # QK_BENCH_SHARED_GPU=1 (testing the multi-rank code path on a one-GPU box): every rank
    # on cuda:0 with a gloo process group.  Never set for a measurement.
    shared_gpu = os.environ.get("QK_BENCH_SHARED_GPU") == "1"
    if shared_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if shared_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        print(f"[bench] rank {rank}/{world}: backend {dist.get_backend()}"
              f"{' nccl ' + '.'.join(map(str, torch.cuda.nccl.version())) if not shared_gpu else ''}"
              f", cuda:{local} {torch.cuda.get_device_name(local)} "
              f"bus {getattr(torch.cuda.get_device_properties(local), 'pci_bus_id', '?')}",
              file=sys.stderr,
              flush=True)
    from paper_2405_02630_b200 import FeatureMapConfig, compute_kernel_matrices, plan_for
    from paper_2405_02630_b200 import device as qdev
    from paper_2405_02630_b200.distributed import KernelJob

    cfg = FeatureMapConfig(N_QUBITS, layers=LAYERS)
    plan = plan_for(cfg)
    info = plan.info
    Atr, Ate = workload_data()
    tr = torch.as_tensor(Atr, device="cuda")
    te = torch.as_tensor(Ate, device="cuda")
    job = KernelJob(plan, N_TRAIN, N_TEST)
    entries = job.layout.entries()

    # Instrument the sweep launches with CUDA events on the launching (current) stream.
    sweep_events = []
    orig = {k: getattr(qdev, k) for k in ("gram", "cross", "gram_into", "cross_into",
                                           "job_into")}

    def timed(fn):
        def wrap(*a, **k):
            s = torch.cuda.current_stream()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            out = fn(*a, **k)
            e1.record(s)
            if recording[0]:
                sweep_events.append((e0, e1))
            return out
        return wrap

    recording = [False]
    for k, fn in orig.items():
        setattr(qdev, k, timed(fn))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def allreduce_scalar(v, op):
        dev_ = "cpu" if dist.get_backend() == "gloo" else "cuda"
        t = torch.tensor([float(v)], device=dev_, dtype=torch.float64)
        dist.all_reduce(t, op=op)
        return float(t.item())

    for _ in range(args.warmup):
        job.run(tr, te)
    barrier()
    clocks = Clocks(local)
    if rank == 0:
        clocks.start()
    barrier()
    recording[0] = True
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(args.steps):
        K_last = job.run(tr, te)
    t1.record()
    torch.cuda.synchronize()
    recording[0] = False
    elapsed = t0.elapsed_time(t1) / 1e3
    if world > 1:
        elapsed = allreduce_scalar(elapsed, dist.ReduceOp.MAX)
    barrier()
    clk = clocks.stop() if rank == 0 else None
    for k, fn in orig.items():
        setattr(qdev, k, fn)

    sweep_s = sum(a.elapsed_time(b) for a, b in sweep_events) / 1e3
    launches_per_step = 2 + len(sweep_events) // max(1, args.steps)
    if world > 1 and rank == 0 and job.placement == "gather":  # unpack launches
        launches_per_step += sum(len(job.layout.segments(r)) for r in range(world))
    value = entries * args.steps / elapsed

    # roofline of the dominant kernel (the pair sweep), per rank, from live CUDA events
    n_sweep = len(sweep_events)
    my_entries = job.layout.rank_entries(rank)  # this rank's cost-balanced tile range
    flops_exec = my_entries * info["flops_per_entry"] * args.steps
    achieved_tf = flops_exec / sweep_s / 1e12 if sweep_s > 0 else None
    props = torch.cuda.get_device_properties(local)
    peaks = {}
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except (OSError, ValueError):
        pass
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    peak_nominal = props.multi_processor_count * 128 * sm_max * 1e6 / 1e12
    peak_dfma = qdev.dfma_peak_flops() / 1e12
    traffic = None
    try:
        tj = json.loads((ROOT / "profiles" / "ncu_traffic.json").read_text())
        traffic = tj.get("sweep_dram_bytes_per_launch")
    except (OSError, ValueError):
        pass
    roofline = {"bound": "fp64", "achieved": achieved_tf, "peak": peak_nominal,
                "unit": "TFLOP/s", "frac": (achieved_tf / peak_nominal) if achieved_tf else None,
                "traffic": traffic,
                "kernel": "qk::sweep_kernel<2,kModeJob,dense,RI=2> (Gram + cross tile list)",
                "flops_per_entry_executed": info["flops_per_entry"],
                "flops_per_entry_algorithmic_F": info["algorithmic_flops_per_entry"],
                "dp_instr_per_entry": info["dp_instr_per_entry"],
                "fp64_pipe_frac": (my_entries * args.steps * info["dp_instr_per_entry"] /
                                   sweep_s / (props.multi_processor_count * 64 * sm_max * 1e6))
                if sweep_s > 0 else None,
                "peak_measured_dfma": peak_dfma,
                "peak_note": "nominal FP64 = SMs x 64 DFMA/clk x 2 x sm_max_mhz (FP64 is not in "
                             "MEASURED_PEAKS.json); peak_measured_dfma = qk_dfma_peak "
                             "microbenchmark in this run",
                "sweep_share_of_step": sweep_s / elapsed if elapsed > 0 else None,
                "sweep_launches": n_sweep, "rank_entries_per_step": my_entries}
    if world > 1 and roofline["frac"] is not None:
        roofline["frac_min_over_ranks"] = allreduce_scalar(roofline["frac"], dist.ReduceOp.MIN)
        roofline["frac_max_over_ranks"] = allreduce_scalar(roofline["frac"], dist.ReduceOp.MAX)

    # e2e through the public API with pinned host buffers (N = 1: the C-ABI host pipeline;
    # N > 1: per-rank H2D + sharded job + gather + D2H on rank 0)
    e2e = None
    if args.e2e_steps > 0:
        h_tr = torch.empty(Atr.shape, dtype=torch.float64, pin_memory=True).numpy()
        h_te = torch.empty(Ate.shape, dtype=torch.float64, pin_memory=True).numpy()
        h_tr[:] = Atr
        h_te[:] = Ate
        h2d = h_tr.nbytes + h_te.nbytes
        d2h = 8 * (N_TRAIN * N_TRAIN + N_TEST * N_TRAIN)
        if world == 1:
            h_K = torch.empty((N_TRAIN, N_TRAIN), dtype=torch.float64, pin_memory=True).numpy()
            h_Kx = torch.empty((N_TEST, N_TRAIN), dtype=torch.float64, pin_memory=True).numpy()
            def e2e_step():
                compute_kernel_matrices(h_tr, h_te, cfg, out_train=h_K, out_test=h_Kx)
        else:
            # every rank drains its row slice of rank 0's matrices into host matrices all
            # ranks map (shared memory, page-locked in each process): N PCIe links in parallel
            out_K, out_Kx = job.host_outputs()

            def e2e_step():
                job.run_host(h_tr, h_te, out_K, out_Kx)
        e2e_step()
        barrier()
        w0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        barrier()
        e_el = time.perf_counter() - w0
        if world > 1:
            e_el = allreduce_scalar(e_el, dist.ReduceOp.MAX)
        e2e = {"value": entries * args.e2e_steps / e_el, "unit": UNIT,
               "h2d_bytes_per_step": int(h2d * (world if world > 1 else 1)),
               "d2h_bytes_per_step": int(d2h), "steps": args.e2e_steps,
               "ms_per_step": 1e3 * e_el / args.e2e_steps,
               "api": "compute_kernel_matrices(train, test) (C-ABI host pipeline "
                      "qk_kernel_matrices_host, pinned buffers)"
               if world == 1 else "KernelJob.run_host (per-rank H2D, sweeps store into rank 0 "
                                  "over NVLink, each rank drains its row slice to shared host "
                                  "memory over its own PCIe link)"}

    # the default public call: pageable numpy in, library-allocated numpy results out (N = 1;
    # the results live in recycled page-locked mappings, kernel_pipeline._HostCache)
    e2e_pageable = None
    if args.e2e_steps > 0 and world == 1:
        compute_kernel_matrices(Atr, Ate, cfg)
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        for _ in range(max(1, args.e2e_steps - 1)):
            compute_kernel_matrices(Atr, Ate, cfg)
        e_el = (time.perf_counter() - w0) / max(1, args.e2e_steps - 1)
        e2e_pageable = {"value": entries / e_el, "unit": UNIT, "ms_per_step": 1e3 * e_el,
                        "steps": max(1, args.e2e_steps - 1),
                        "h2d_bytes_per_step": int(Atr.nbytes + Ate.nbytes),
                        "d2h_bytes_per_step": int(8 * (N_TRAIN * N_TRAIN + N_TEST * N_TRAIN)),
                        "api": "compute_kernel_matrices(train, test, cfg): pageable numpy in, "
                               "library-allocated numpy results out (a new array per call, "
                               "backed by a recycled page-locked mapping)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_run(Atr, Ate, args.cpu_seconds)
        cpu.pop("seconds", None)
        ref, got = reference_python_run(Atr, Ate)
        if got is not None:
            pairs, amp = got
            K, Kx = (k.cpu().numpy() for k in K_last)
            ours = np.where(pairs[:, 0] < N_TRAIN, K[np.minimum(pairs[:, 0], N_TRAIN - 1),
                                                     pairs[:, 1]],
                            Kx[np.maximum(pairs[:, 0] - N_TRAIN, 0), pairs[:, 1]])
            ref["parity_vs_this_run"] = parity_vs_reference(Atr, Ate, pairs, amp, ours)
        cpu["reference_python"] = ref

    launches_total = launches_per_step * args.steps
    if world > 1:
        launches_total = allreduce_scalar(launches_total, dist.ReduceOp.SUM)
    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup,
               "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
               "config": dict(WORKLOAD, parallelism=f"tile-sharded x{world}",
                              entries_per_step=entries),
               "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
               "e2e_pageable": e2e_pageable, "clocks": clk,
               "gpu_launches": int(launches_total),
               "gpu": props.name, "plan": info}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
