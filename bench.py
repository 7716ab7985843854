#!/usr/bin/env python
"""Benchmark of the B200-native batched forward-dynamics path.

Metric (BASELINE.json): FD solves/sec (batch, n links, FP64) per algorithm;
% of HBM/FP64 roofline. Headline workload at N=1 is configs[1]:
ABIA on 65,536 independent chains x 32 links with random q/qd/tau (the
reference's seeded generators, seed 42). Under torchrun each rank solves its
own 65,536 chains (weak scaling, no collective on the hot path).

  value    device-resident inputs, K steps of pd_forward_dynamics_device timed
           with CUDA events on the launch stream, max over ranks
  e2e      same metric through the public host API (pd_forward_dynamics via
           paper_1609_06779_b200.Context.solve) with pinned host buffers: H2D
           of q/qdot/tau and D2H of qddot + slot status inside every step
  roofline algorithmic bytes / flops of the frozen work model (SURVEY.md §8d:
           B_alg = 256 n bytes, F_alg(ABIA) = 1400 n flops per solve) over the
           kernel's average launch time
  cpu_baseline  the CPU restatement of the reference path (oracle/, OpenMP over
           all host cores) on a bounded sample of the same workload

`--impl reference` times the reference's CPU path (the oracle port, since the
reference itself cannot be compiled in this image) on the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FD solves/sec (batch, n links, FP64) per algorithm; % of HBM/FP64 roofline"
UNIT = "solves/s"


def f_alg(algo: str, n: int) -> float:
    """Frozen algorithmic flops per solve (FMA = 2)."""
    L = 0
    while (1 << L) < n:
        L += 1
    if algo == "abia":
        return 1400.0 * n
    if algo == "jsiia":
        return 482.0 * n + 102.0 * n * n + n ** 3 / 3.0
    return 2833.0 * n + 1200.0 * (n * L - (1 << L) + 1)


def b_alg(n: int, shared: bool) -> float:
    """Frozen algorithmic bytes per solve: 28 model doubles + q, qd, tau, qdd per link."""
    return (32.0 if shared else 256.0) * n


WORKLOADS = {
    "c1": dict(desc="configs[0]: ABIA, 8-link chain, 1024 random states (shared model)", algo="abia", n=8,
               batch=1024, shared=True),
    "c2": dict(desc="configs[1]: ABIA, 65,536 chains x 32 links, random q/qd/tau", algo="abia", n=32, batch=65536,
               shared=False),
    "c2j": dict(desc="configs[1]: JSIIA, 65,536 chains x 32 links, random q/qd/tau", algo="jsiia", n=32,
                batch=65536, shared=False),
    "c3": dict(desc="configs[2]: CFA via OEE, 4,096 chains x 256 links", algo="cfa", n=256, batch=4096,
               shared=False),
    "c4a": dict(desc="configs[3]: single chain, 1,024 links (ABIA, latency)", algo="abia", n=1024, batch=1,
                shared=False),
    "c4c": dict(desc="configs[3]: single chain, 1,024 links (CFA, latency)", algo="cfa", n=1024, batch=1,
                shared=False),
    "c4j": dict(desc="configs[3]: single chain, 1,024 links (JSIIA, latency)", algo="jsiia", n=1024, batch=1,
                shared=False),
    # configs[4]: the global batch is fixed and sharded over the ranks (strong scaling)
    "c5a": dict(desc="configs[4]: ABIA, 1M chains x 64 links, batch-sharded", algo="abia", n=64, batch=1 << 20,
                shared=False, sharded=True),
    "c5j": dict(desc="configs[4]: JSIIA, 1M chains x 64 links, batch-sharded", algo="jsiia", n=64, batch=1 << 20,
                shared=False, sharded=True),
    "c5c": dict(desc="configs[4]: CFA, 1M chains x 64 links, batch-sharded", algo="cfa", n=64, batch=1 << 20,
                shared=False, sharded=True),
}


def local_batch(wl: dict, world: int, rank: int):
    """(first problem, count) this rank solves: sharded configs split the
    global batch (sharding.shard_bounds), the others give every rank a full
    batch of its own chains (weak scaling)."""
    if wl.get("sharded"):
        from paper_1609_06779_b200.sharding import shard_bounds
        lo, hi = shard_bounds(wl["batch"], world, rank)
        return lo, hi - lo
    return rank * wl["batch"], wl["batch"]


# ----------------------------------------------------------------------------- helpers
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the GPU works."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-i", str(self.dev),
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (FileNotFoundError, OSError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(self.NAMES, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        load = [s for s in sm if s > 500] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup():
    """One rank per GPU over NCCL. With more ranks than visible GPUs (a
    multi-process check on a one-GPU box) ranks share devices round-robin and
    the control collectives (barrier, max of the timings, gather) run on gloo."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        ndev = max(1, torch.cuda.device_count())
        if world <= ndev:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            local = local % ndev
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
    return world, rank, local


def _on_nccl() -> bool:
    import torch.distributed as dist
    return dist.get_backend() == "nccl"


def dist_max(x: float, world: int, local: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}" if _on_nccl() else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def dist_barrier(world: int, local: int):
    if world > 1:
        import torch.distributed as dist
        if _on_nccl():
            dist.barrier(device_ids=[local])
        else:
            dist.barrier()


# ----------------------------------------------------------------------------- CPU arm
def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_reference(algo: str, n: int, links, q, qd, tau, budget_s: float, reps: int, warm: int):
    """Times the CPU restatement of the reference path (oracle/) on the
    largest prefix of the workload that keeps reps+warm calls within budget_s.
    Returns (solves/s, sample size, cores, oracle qdd of the sample)."""
    from oracle import pyoracle as po
    cores = po.lib().orc_num_threads()
    if isinstance(links, DeviceChains):  # device-generated chains: time a host-generated prefix
        links = links.host_prefix(8192)
        q, qd, tau = q[:len(links)], qd[:len(links)], tau[:len(links)]
    probe = min(len(q), 512 if algo != "jsiia" else 128)
    t0 = time.perf_counter()
    po.batch_forward_dynamics(algo, links[:probe], [0, 0, -9.81], q[:probe], qd[:probe], tau[:probe])
    rate = probe / max(time.perf_counter() - t0, 1e-6)
    S = int(max(64, min(len(q), rate * budget_s / max(reps + warm, 1))))
    ls = links if links.shape[0] == 1 else links[:S]
    for _ in range(warm):
        po.batch_forward_dynamics(algo, ls, [0, 0, -9.81], q[:S], qd[:S], tau[:S])
    t0 = time.perf_counter()
    for _ in range(reps):
        ref, _ = po.batch_forward_dynamics(algo, ls, [0, 0, -9.81], q[:S], qd[:S], tau[:S])
    dt = time.perf_counter() - t0
    return S * reps / dt, S, cores, ref


class DeviceChains:
    """A rank's slice [g0, g0 + count) of a cell's chains, generated, validated
    and packed on the device (pd_set_models_workload): no host model buffer
    (15.5 GiB at c5). host_prefix() gives the first chains on the host for the
    CPU baseline / parity sample."""

    def __init__(self, cell: int, n: int, g0: int, count: int):
        self.cell, self.n, self.g0, self.count = cell, n, g0, count
        self.shape = (count, n, 31)

    def host_prefix(self, k: int):
        from paper_1609_06779_b200 import workload as W
        return W.workload_chains(self.cell, self.n, min(k, self.count), g0=self.g0)


def gen_workload(wl: dict, rank: int, world: int = 1):
    from paper_1609_06779_b200 import workload as W
    n, B = wl["n"], wl["batch"]
    cell = W.workload_seed(42, n, B)
    if wl.get("sharded"):
        lo, cnt = local_batch(wl, world, rank)
        inputs = tuple(np.ascontiguousarray(a[lo:lo + cnt]) for a in W.workload_inputs(cell, n, B, 0))
        return DeviceChains(cell, n, lo, cnt), inputs, None
    if wl["shared"]:
        links = W.workload_chains(cell, n, 1)
        qs = [W.workload_inputs(cell, n, 1, r) for r in range(B)]
        q = np.concatenate([x[0] for x in qs])
        qd = np.concatenate([x[1] for x in qs])
        tau = np.concatenate([x[2] for x in qs])
        return links, (q, qd, tau), None
    links = W.workload_chains(cell, n, B, g0=rank * B)
    inputs = W.workload_inputs(cell, n, B, 0)
    inputs2 = W.workload_inputs(cell, n, B, 1)
    return links, inputs, inputs2


def oracle_workload(wl: dict):
    """The same workload as gen_workload, generated by the oracle's restatement
    of the reference generators (bench.cpp:350-383, model.cpp:157-185), so the
    reference arm maps only oracle/build/liboracle.so."""
    from oracle import pyoracle as po
    n, B = wl["n"], wl["batch"]
    cell = po.workload_seed(42, n, B)
    if wl["shared"]:
        links = po.workload_chains(cell, n, 1)
        qs = [po.workload_inputs(cell, n, 1, r) for r in range(B)]
        return links, tuple(np.concatenate([x[k] for x in qs]) for k in range(3))
    return None, (cell, n, B)


def run_reference_arm(args, wl):
    world, rank, _ = (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
                      int(os.environ.get("LOCAL_RANK", "0")))
    if rank != 0:
        return
    from oracle import pyoracle as po
    cores = po.lib().orc_num_threads()
    algo, n = wl["algo"], wl["n"]
    links, spec = oracle_workload(wl)
    if links is None:  # independent chains: generate the prefix the CPU can time
        cell, _, B = spec
        probe_links = po.workload_chains(cell, n, min(B, 256))
        q, qd, tau = po.workload_inputs(cell, n, B, 0)
    else:
        probe_links = links
        q, qd, tau = spec
    # bound the whole --steps/--warmup run to ~90 s of CPU work
    probe = min(len(q), 256)
    t0 = time.perf_counter()
    po.batch_forward_dynamics(algo, probe_links if wl["shared"] else probe_links[:probe], [0, 0, -9.81], q[:probe],
                              qd[:probe], tau[:probe])
    rate = probe / max(time.perf_counter() - t0, 1e-6)
    S = int(max(32, min(len(q), rate * 90.0 / max(args.steps + args.warmup, 1))))
    ls = links if wl["shared"] else po.workload_chains(spec[0], n, S)
    for _ in range(args.warmup):
        po.batch_forward_dynamics(algo, ls, [0, 0, -9.81], q[:S], qd[:S], tau[:S])
    t0 = time.perf_counter()
    for _ in range(args.steps):
        po.batch_forward_dynamics(algo, ls, [0, 0, -9.81], q[:S], qd[:S], tau[:S])
    dt = time.perf_counter() - t0
    value = S * args.steps / dt
    sample = (f"first {S} of {wl['batch']} problems of {args.workload} per step "
              f"(reference CPU path restated in oracle/, OpenMP dynamic over {cores} threads; {cpu_model()})")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong" if wl.get("sharded") else "weak", "vs_baseline": None, "dtype": "f64",
        "data": DATA,
        "config": workload_config(args.workload, wl, wl["batch"], wl["batch"] * (1 if wl.get("sharded") else world),
                                  world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


DATA = "synthetic: reference generators workload_chains/workload_inputs (seed 42), random-init chains"


def workload_config(name: str, wl: dict, batch_per_gpu: int, global_batch: int, world: int) -> dict:
    """The `config` object both arms print (same keys and values)."""
    return {"workload": f"{name}: {wl['desc']}", "algo": wl["algo"], "n_links": wl["n"],
            "batch_per_gpu": batch_per_gpu, "global_batch": global_batch, "parallelism": f"batch-sharded x{world}",
            "l2": "inputs larger than L2 (%.0f MB streamed per step)" % (b_alg(wl["n"], wl["shared"]) * batch_per_gpu
                                                                        / 1e6)
            if b_alg(wl["n"], wl["shared"]) * batch_per_gpu > 126e6 else "L2 not flushed (small workload)"}


# ----------------------------------------------------------------------------- GPU arm
def time_device(ctx, algo, B, n, dev_inputs, steps, warmup, stream):
    """Device-resident timed loop; returns (ms total, launches in region)."""
    import torch
    from paper_1609_06779_b200 import FdAlgo
    qdd = torch.empty((n, B), dtype=torch.float64, device=dev_inputs[0][0].device)
    st = torch.empty((3, B), dtype=torch.int32, device=qdd.device)

    def step(k):
        q, qd, tau = dev_inputs[k % len(dev_inputs)]
        ctx.solve_device(FdAlgo[algo], B, q.data_ptr(), qd.data_ptr(), tau.data_ptr(), qdd.data_ptr(),
                         st[0].data_ptr(), st[1].data_ptr(), st[2].data_ptr())

    for k in range(warmup):
        step(k)
    torch.cuda.synchronize()
    l0 = ctx.kernel_launches()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(steps):
        step(k)
    e1.record(stream)
    torch.cuda.synchronize()
    bad = int((st[0] != 0).sum().item())
    if bad:
        raise RuntimeError(f"{bad} slots reported errors in the timed loop")
    return e0.elapsed_time(e1), ctx.kernel_launches() - l0, qdd


def qdd_for_first_inputs(ctx, algo, B, n, dev_inputs, qdd, steps):
    """Host copy ([link][problem]) of the qdd the timed loop computed for the
    first input set (re-solved untimed if the last step used another set)."""
    import torch
    from paper_1609_06779_b200 import FdAlgo
    if (steps - 1) % len(dev_inputs) != 0:
        q, qd, tau = dev_inputs[0]
        ctx.solve_device(FdAlgo[algo], B, q.data_ptr(), qd.data_ptr(), tau.data_ptr(), qdd.data_ptr())
        ctx.synchronize()
    torch.cuda.synchronize()
    return qdd.cpu().numpy()


def measure_workload(ctx, name, wl, steps, warmup, rank, local, stream, want_e2e, e2e_steps, world=1):
    import torch
    n, algo = wl["n"], wl["algo"]
    links, inp, inp2 = gen_workload(wl, rank, world)
    B = len(inp[0])
    if isinstance(links, DeviceChains):
        ms, mr = ctx.set_models_workload(links.cell, n, links.count, g0=links.g0)
    else:
        ms, mr = ctx.set_models(links, None)
    assert (ms == 0).all()
    dev = torch.device("cuda", local)

    def to_dev(x):
        return torch.from_numpy(np.ascontiguousarray(x.T)).to(dev)  # [link][problem]

    dev_inputs = [tuple(to_dev(a) for a in inp)]
    if inp2 is not None:
        dev_inputs.append(tuple(to_dev(a) for a in inp2))
    ms_total, launches, qdd = time_device(ctx, algo, B, n, dev_inputs, steps, warmup, stream)
    res = {"ms_total": ms_total, "launches": launches, "links": links, "inputs": inp, "B": B,
           "variant": ctx.last_variant(),
           # qdd of the last timed step (inputs set len(dev_inputs) - 1 ... wrap): keep the one matching inp
           "qdd": qdd_for_first_inputs(ctx, algo, B, n, dev_inputs, qdd, steps)}
    if want_e2e:
        pin = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in inp]
        out = torch.empty((B, n), dtype=torch.float64).pin_memory()
        args = [p.numpy() for p in pin]
        from paper_1609_06779_b200 import FdAlgo
        slots = tuple(np.zeros(B, np.int32) for _ in range(3))  # the caller's slot arrays, reused per step
        for _ in range(2):
            ctx.solve(FdAlgo[algo], *args, out=out.numpy(), status_out=slots)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            _, st, _, _ = ctx.solve(FdAlgo[algo], *args, out=out.numpy(), status_out=slots)
        dt = time.perf_counter() - t0
        assert (st == 0).all()
        res["e2e_s"] = dt
        res["e2e_steps"] = e2e_steps
        res["h2d"] = 3 * B * n * 8
        # qddot, plus the 4-byte OR of the slot codes: when every slot succeeded
        # (asserted above) the per-slot arrays are zero-filled on the host
        # instead of copied (capi.cu host_forward_dynamics)
        res["d2h"] = B * n * 8 + 4
    return res


# ncu --set full captures of the dominant kernel per workload (profiles/, same
# kernel and config as the bench command): DRAM bytes per launch
NCU_TRAFFIC = {"c2": "profiles/ncu_c2_r2d.txt", "c3": "profiles/ncu_c3_r2f.txt",
               "c2j": "profiles/ncu_c2j_r2c.txt", "c5j": "profiles/ncu_c5j_r2b.txt",
               "c5c": "profiles/ncu_c5c_r2e.txt"}


def dropin_api_timings():
    """The reference's own call paths timed through the C++ drop-in
    (libpardyn.so): pardyn_bench --mode link (forward_dynamics on one chain,
    host vectors in and out, the model re-sent every call as the reference
    API does) for the c4 chain, and --mode group (batch_forward_dynamics over
    FdProblem values) for c2. Steady-clock means of the harness
    (bench.cpp:150-278 semantics)."""
    import csv
    import subprocess
    import tempfile
    exe = os.path.join(ROOT, "paper_1609_06779_b200", "lib", "pardyn_bench")
    if not os.path.exists(exe):
        return None
    out = {}
    with tempfile.TemporaryDirectory() as d:
        runs = {"c4": ["--mode", "link", "--algos", "abia,cfa,jsiia", "--links", "1024", "--repeats", "100"],
                "c2": ["--mode", "group", "--algos", "abia,jsiia", "--links", "32", "--groups", "65536",
                       "--repeats", "5"]}
        for tag, argv in runs.items():
            path = os.path.join(d, tag + ".csv")
            r = subprocess.run([exe, *argv, "--out", path], capture_output=True, text=True, timeout=900)
            if r.returncode != 0:
                out[tag] = {"error": (r.stderr or r.stdout)[-300:]}
                continue
            for row in csv.DictReader(open(path)):
                g = int(row["n_groups"])
                key = f"{tag}_{row['algo']}"
                out[key] = {"call": "forward_dynamics" if g == 1 else "batch_forward_dynamics",
                            "n_links": int(row["n_links"]), "problems_per_call": g,
                            "mean_us": float(row["mean_us"]), "stddev_us": float(row["stddev_us"]),
                            "solves_per_s": g / (float(row["mean_us"]) * 1e-6), "repeats": int(row["repeats"])}
    return out


def ncu_traffic(workload: str):
    """dram__bytes_read.sum + dram__bytes_write.sum of the committed capture, or None."""
    path = os.path.join(ROOT, NCU_TRAFFIC.get(workload, ""))
    if workload not in NCU_TRAFFIC or not os.path.exists(path):
        return None
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    got = {}
    for line in open(path):  # first occurrence of each (summaries may repeat a metric in a later section)
        parts = line.split()
        if len(parts) >= 3 and parts[0] in ("dram__bytes_read.sum", "dram__bytes_write.sum") and parts[0] not in got:
            got[parts[0]] = float(parts[1]) * scale.get(parts[2], 1.0)
    return {"bytes_per_launch": sum(got.values()), "source": NCU_TRAFFIC[workload]} if len(got) == 2 else None


def _executed_fp64():
    try:
        with open(os.path.join(ROOT, "profiles", "executed_fp64_r2.json")) as f:
            return json.load(f)
    except OSError:
        return {}


EXECUTED_FP64 = _executed_fp64()


def roofline_entry(wl, ms_per_step, bw_gbs, fp64_tflops, traffic=None):
    """Algorithmic work of one step (the whole batch) over the step's device
    time. A step is one launch for the batched kernels; multi-kernel paths
    (tau_delta pre-pass, cooperative long-chain pipelines, chunked global-
    workspace launches) count all their kernels."""
    n, B, algo = wl["n"], wl["batch"], wl["algo"]
    bytes_ = b_alg(n, wl["shared"]) * B
    flops = f_alg(algo, n) * B
    t = ms_per_step * 1e-3
    gbs = bytes_ / t / 1e9
    tfl = flops / t / 1e12
    t_hbm = bytes_ / (bw_gbs * 1e9)
    t_fp = flops / (fp64_tflops * 1e12)
    hbm = {"bound": "hbm", "achieved": gbs, "peak": bw_gbs, "unit": "GB/s", "frac": gbs / bw_gbs, "traffic": traffic,
           "algorithmic_bytes": bytes_}
    fp = {"achieved": tfl, "peak": fp64_tflops, "unit": "TFLOP/s (FP64)", "frac": tfl / fp64_tflops,
          "flops_per_solve_algorithmic": f_alg(algo, n)}
    ex = EXECUTED_FP64.get(wl.get("name", ""))
    if ex:  # the FP64 work the kernel actually executes (ncu SASS counts), beside the frozen F_alg
        fp["flops_per_solve_executed"] = ex["flops_per_solve"]
        fp["frac_executed"] = ex["flops_per_solve"] * B / t / 1e12 / fp64_tflops
        fp["executed_source"] = ex["source"]
    binding = "hbm" if t_hbm >= t_fp else "fp64"
    return hbm, fp, binding, {"bytes_per_launch": bytes_, "flops_per_launch": flops,
                              "roofline_frac": (max(t_hbm, t_fp) / t)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=200)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c2")
    ap.add_argument("--no-extra", action="store_true", help="skip the per-algorithm side measurements")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference_arm(args, wl)
        return

    world, rank, local = dist_setup()
    import torch
    torch.cuda.set_device(local)
    from paper_1609_06779_b200 import Context
    ctx = Context(local)
    # a dedicated (non-default) stream: the kernels and the timing events
    # must live on the same stream
    stream = torch.cuda.Stream(device=local)
    ctx.set_stream(stream.cuda_stream)

    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass
    bw = float(peaks.get("hbm_gbs", 6650.0))
    bw_src = "measured (MEASURED_PEAKS.json)" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"
    fp64_peak = ctx.probe_fp64_peak()

    sampler = ClockSampler(local)
    sampler.start()
    dist_barrier(world, local)
    torch.cuda.synchronize()
    res = measure_workload(ctx, args.workload, wl, args.steps, args.warmup, rank, local, stream, not args.no_e2e,
                           e2e_steps=max(3, min(args.steps, 30)), world=world)
    clocks = sampler.stop()
    ms_max = dist_max(res["ms_total"], world, local)
    e2e_max = dist_max(res.get("e2e_s", 0.0), world, local)

    n, B = wl["n"], res["B"]
    sharded = bool(wl.get("sharded"))
    global_batch = wl["batch"] if sharded else B * world
    total = global_batch * args.steps
    value = total / (ms_max * 1e-3)
    ms_per_step = ms_max / args.steps
    # roofline of this rank's step on its own (local) batch
    tr = ncu_traffic(args.workload) if world == 1 else None
    hbm, fp, binding, work = roofline_entry(dict(wl, batch=B, name=args.workload), res["ms_total"] / args.steps, bw,
                                            fp64_peak,
                                            traffic=tr["bytes_per_launch"] if tr else None)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64",
        "data": DATA,
        "config": workload_config(args.workload, wl, B, global_batch, world),
        "roofline": hbm,
        "roofline_traffic_source": (tr["source"] + " (ncu --set full, DRAM read + write bytes per launch)") if tr
        else None,
        "roofline_fp64": fp,
        "roofline_binding": binding,
        "roofline_frac_of_binding": work["roofline_frac"],
        "peaks": {"hbm_gbs": bw, "hbm_source": bw_src, "fp64_tflops_measured": fp64_peak},
        "gpu_launches": res["launches"],
        "clocks": clocks,
    }
    import torch
    if world > max(1, torch.cuda.device_count()):
        line["note"] = (f"{world} ranks share {torch.cuda.device_count()} device(s): a multi-process correctness check "
                        f"of the sharded path, not a scaling measurement")
    if "e2e_s" in res:
        line["e2e"] = {"value": global_batch * res["e2e_steps"] / e2e_max, "unit": UNIT,
                       "h2d_bytes_per_step": res["h2d"] * world, "d2h_bytes_per_step": res["d2h"] * world,
                       "timing": "wall clock around pd_forward_dynamics (pinned host buffers), max over ranks"}

    if rank == 0 and world == 1 and not args.no_cpu:
        q, qd, tau = res["inputs"]
        v, S, cores, ref = cpu_reference(wl["algo"], n, res["links"], q, qd, tau, budget_s=12.0, reps=5, warm=1)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "cpu_model": cpu_model(),
                                "sample": f"first {S} problems of {args.workload}, 1 warm-up + 5 timed whole-batch "
                                          f"calls, reference CPU path restated in oracle/ (OpenMP dynamic)"}
        # the checker, outside every timed region: the timed loop's qdd of the
        # sampled problems against the oracle's (rel_gap, oracles.hpp:64-66)
        got = res["qdd"][:, :S].T if res["qdd"].shape[1] >= S else None
        if got is not None:
            gaps = np.linalg.norm(got - ref, axis=1) / np.maximum(1.0, np.linalg.norm(ref, axis=1))
            line["parity"] = {"max_rel_gap": float(gaps.max()), "tolerance": 1e-9, "slots": int(S),
                              "ok": bool(gaps.max() <= 1e-9), "against": "oracle/ (CPU restatement)"}

    if rank == 0 and world == 1 and not args.no_extra:
        extra = {}
        for name in ("c2j", "c3", "c1", "c4a", "c4c", "c4j", "c5a", "c5j", "c5c"):
            if name == args.workload:
                continue
            w = WORKLOADS[name]
            steps = 3 if w["batch"] == 1 or w.get("sharded") else 20
            r = measure_workload(ctx, name, w, steps, 3, 0, local, stream, False, 0)
            mps = r["ms_total"] / steps
            h, f, b, wk = roofline_entry(dict(w, name=name), mps, bw, fp64_peak)
            extra[name] = {"workload": w["desc"], "solves_per_s": w["batch"] * steps / (r["ms_total"] * 1e-3),
                           "ms_per_step": mps, "hbm_frac": h["frac"], "fp64_frac": f["frac"],
                           "fp64_frac_executed": f.get("frac_executed"), "binding": b,
                           "roofline_frac_of_binding": wk["roofline_frac"]}
        dropin = dropin_api_timings()
        if dropin:
            extra["dropin_api"] = dropin
        line["extra"] = extra

    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
