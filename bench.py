#!/usr/bin/env python
"""SAMO step benchmark (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload gpt-2.7b] [--sparsity 0.9]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N   (N > 1)
    python bench.py --impl reference ...      (the reference's CPU implementation)

One step = one pass of the SAMO per-step parameter-state path over one batch of
synthetic dense gradients.  N = 1: K1 gather (+unscale/cast) -> K23 Adam +
downcast + expand.  N > 1 (data parallel, each rank its own gradient batch):
the default exchange is fused over NVLink peer memory — K1 ->
shard update (every rank's binary16 grads summed in rank order, Adam on the
rank's 1/N shard, binary16 weights stored to every rank) -> expand; NCCL
carries only two tiny allreduces that double as barriers.  The per-GPU
workload (the full GPT set) is fixed as N grows ("scaling": "weak") and
`value` is N * phi / t_step (dense parameters stepped per second, whole job).

Rank 0 prints ONE JSON line.  All timing is CUDA events on the launching
stream; multi-GPU times are the max over ranks.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "SAMO step params/sec (gather+allreduce+Adam+expand); HBM & bus GB/s vs peak"
UNIT = "params/s"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["samo", "reference"], default="samo")
    ap.add_argument("--workload", default="gpt-2.7b")
    ap.add_argument("--sparsity", type=float, default=0.9)
    ap.add_argument("--tile", type=int, default=0, help="dense elements per tile (0 = default)")
    ap.add_argument("--seed", type=int, default=1234)
    ap.add_argument("--grad-dtype", choices=["f16", "bf16"], default="f16",
                    help="dense gradient type (bf16: north_star's other 16-bit type; no CPU reference)")
    ap.add_argument("--e2e-steps", type=int, default=0, help="0 = min(steps, 10)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-fused", action="store_true",
                    help="skip the side probes (fused dW-GEMM sink, FC-layer sweep of config 2)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-blocks", type=int, default=0, help="GPT blocks in the CPU sample")
    ap.add_argument("--cpu-wte-rows", type=int, default=4096,
                    help="rows of the token embedding in the CPU sample")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no e2e/CPU legs)")
    ap.add_argument("--graph", action="store_true",
                    help="time whole steps launched as one CUDA graph (small, launch-bound configs); "
                         "per-kernel times come from a separate staged pass")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# helpers

def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "bf16_tflops": float(d.get("bf16_tflops", 0)) or None,
                "src": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 2250.0, "src": "fallback"}


class ClockSampler:
    """SM / memory clocks and throttle reasons of rank 0's GPU through NVML
    in-process (the nvidia_ml_py binding): clocks and reasons just before the
    timed region and just after it; in it, the clocks right after its steps
    are queued (the GPU is then still running them) and every 0.5 s.  Every clock query stalls
    the GPU for a few ms, which the tightly coupled data-parallel step pays on
    every rank: at N = 4 over 50 steps, 2.82-2.85 ms unsampled against
    2.95-3.57 ms with a 100 ms NVML sampler, 2.87-3.08 with one nvidia-smi per
    rank at 100 ms and 4.07-4.28 with one nvidia-smi over all GPUs at 200 ms
    (profiles/r02z_n4_sampler_*.log).  SAMO_BENCH_CLOCKS: nvml
    (default), smi (nvidia-smi at 100 ms, for A/B), nvml_sm / nvml_reasons /
    nvml_power (query subsets), off."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,clocks.mem")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.mode = os.environ.get("SAMO_BENCH_CLOCKS", "nvml")
        self.proc = None
        self.lines: list[str] = []          # nvidia-smi rows (smi mode)
        self.samples: list[tuple] = []      # (sm, sm_max, mem, power or None, reasons)
        self._stop = threading.Event()
        self._t = None
        self.in_region = 0

    def __len__(self):
        return len(self.samples) + len(self.lines)

    # -- NVML in-process ------------------------------------------------------
    def _nvml_sample(self, with_reasons: bool = True):
        import pynvml as N
        h = self._h
        reasons = set()
        if with_reasons and self.mode != "nvml_sm":
            bits = N.nvmlDeviceGetCurrentClocksEventReasons(h)
            flags = (N.nvmlClocksEventReasonHwSlowdown, N.nvmlClocksEventReasonHwThermalSlowdown,
                     N.nvmlClocksEventReasonSwThermalSlowdown, N.nvmlClocksEventReasonSwPowerCap)
            reasons = {nm for nm, f in zip(self.NAMES, flags) if bits & f}
        power = N.nvmlDeviceGetPowerUsage(h) / 1000.0 if self.mode == "nvml_power" else None
        sm = float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)) if self.mode != "nvml_reasons" else self._max
        mem = float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_MEM)) if self.mode == "nvml" else None
        self.samples.append((sm, self._max, mem, power, reasons))

    def sample_now(self):
        """One clock sample now (call once the timed steps are queued).  The
        throttle-reason query stalls the GPU longest, so in-region samples
        read the clocks only; the reasons come from the samples taken just
        before and just after the region."""
        if self._t is not None and self.mode.startswith("nvml"):
            try:
                self._nvml_sample(with_reasons=False)
                self.in_region += 1
            except Exception:  # noqa: BLE001
                pass

    def _nvml_loop(self):
        while not self._stop.wait(0.5):
            try:
                self._nvml_sample(with_reasons=False)
            except Exception:  # noqa: BLE001  (a failed read only loses a sample)
                pass

    def __enter__(self):
        if self.gpu is None or self.mode == "off":
            return self
        if self.mode.startswith("nvml"):
            try:
                import pynvml as N
                N.nvmlInit()
                self._h = N.nvmlDeviceGetHandleByIndex(int(self.gpu))
                self._max = float(N.nvmlDeviceGetMaxClockInfo(self._h, N.NVML_CLOCK_SM))
                self._nvml_sample()  # NVML is up before the caller starts its clock
                self._t = threading.Thread(target=self._nvml_loop, daemon=True)
                self._t.start()
            except Exception:  # noqa: BLE001  (no NVML: no clocks)
                self._t = None
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", self.gpu, f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            # nvidia-smi's start-up: let it finish (first sample in) before the
            # caller starts its clock
            t_end = time.perf_counter() + 3.0
            while not self.lines and self.proc.poll() is None and time.perf_counter() < t_end:
                time.sleep(0.01)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def active(self) -> bool:
        return self._t is not None

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None and self.mode.startswith("nvml"):
            self._t.join(timeout=1.0)
            try:
                self._nvml_sample()  # reasons right after the region
            except Exception:  # noqa: BLE001
                pass
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        elif self._t is not None:
            self._t.join(timeout=1.0)

    def summary(self) -> dict:
        rows = list(self.samples)
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm, mx = float(parts[0]), float(parts[1])
            except ValueError:
                continue
            reasons = {nm for nm, v in zip(self.NAMES, parts[3:7]) if v.lower().startswith("active")}
            vals = []
            for v in (parts[7] if len(parts) > 7 else "", parts[2]):
                try:
                    vals.append(float(v))
                except ValueError:
                    vals.append(None)
            rows.append((sm, mx, vals[0], vals[1], reasons))
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "source": self.mode}
        out = {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
               "reasons": sorted(set().union(*(r[4] for r in rows))), "samples": len(rows),
               "source": f"{self.mode}, rank 0's GPU", "samples_in_region": self.in_region}
        mem = [r[2] for r in rows if r[2] is not None]
        pw = [r[3] for r in rows if r[3] is not None]
        if mem:
            out["mem_mhz"] = statistics.median(mem)
        if pw:
            out["power_w_max"] = max(pw)
        return out


def gpt_blocks_of(wl):
    """Indices of tensors grouped per transformer block (for CPU samples)."""
    blocks = {}
    for i, t in enumerate(wl.tensors):
        key = t.name.split(".")[0] if t.name.startswith("h") else "_other"
        blocks.setdefault(key, []).append(i)
    return [v for k, v in blocks.items() if k != "_other"] or [list(range(len(wl.tensors)))]


def partition(sizes, nbins):
    """Greedy LPT partition of item indices into nbins by size."""
    order = sorted(range(len(sizes)), key=lambda i: -sizes[i])
    bins = [[] for _ in range(nbins)]
    load = [0] * nbins
    for i in order:
        b = load.index(min(load))
        bins[b].append(i)
        load[b] += sizes[i]
    return [sorted(b) for b in bins if b]


def piece_cost(dense: int, kept: int) -> float:
    """Relative CPU cost of the reference step on one layer: the dense passes
    (sink gather read, theta16 zero-fill + expand) scale with dense_len, the
    software half conversions, unscale and Adam with the kept count."""
    return dense + 3.0 * kept


def split_layers(dense_len, idx_sets, theta_sets, grad_sets, threads, per_thread=4):
    """Element-range pieces of the layers for `threads` balanced trainers.

    Every step operation of the reference is per element (sink gather,
    unscale, Adam, downcast + expand), so a layer cut into contiguous dense
    ranges [d0, d1) — indices rebased to d0, the matching theta32 range, the
    dense gradient slice — does exactly the work of the whole layer.  Layers
    are cut until no piece costs more than 1/(per_thread * threads) of the
    total, then the pieces are LPT-partitioned over the threads.  Returns
    (pieces, parts, balance = max thread load / mean thread load)."""
    import numpy as np
    total = sum(piece_cost(d, len(i)) for d, i in zip(dense_len, idx_sets))
    target = total / max(1, threads * per_thread)
    pieces = []
    for d, idx, th, g in zip(dense_len, idx_sets, theta_sets, grad_sets):
        k = max(1, int(np.ceil(piece_cost(d, len(idx)) / target))) if threads > 1 else 1
        bounds = [d * j // k for j in range(k + 1)]
        for d0, d1 in zip(bounds, bounds[1:]):
            if d1 <= d0:
                continue
            a, b = np.searchsorted(idx, d0), np.searchsorted(idx, d1)
            pieces.append((d1 - d0, (idx[a:b] - np.uint32(d0)).astype(np.uint32), th[a:b], g[d0:d1]))
    costs = [piece_cost(p[0], len(p[1])) for p in pieces]
    parts = partition(costs, min(threads, len(pieces)))
    loads = [sum(costs[i] for i in part) for part in parts]
    return pieces, parts, max(loads) / (sum(loads) / len(loads))


def cpu_reference_sample(dense_len, idx_sets, theta_sets, grad_sets, cfg_vals, reps, warm=1,
                         threads=None):
    """Times the UNMODIFIED reference (oracle/_ref) step — sink gather +
    SamoTrainer::optimizer_step — on host threads (SURVEY §8(d) CPU
    baseline).  threads = 1 is the reference as shipped: one trainer over the
    layers as they are.  threads = T > 1 (default: every CPU this process may
    use): the layers cut into balanced element ranges (split_layers) over T
    independent trainers.  Returns {sec, threads, balance, pieces}."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle.oracle import Cfg, RefLib, RefSession
    ref = RefLib()
    cfg = Cfg(*cfg_vals)
    T = threads or len(os.sched_getaffinity(0))
    pieces, parts, balance = split_layers(dense_len, idx_sets, theta_sets, grad_sets, T)
    sessions = []
    for part in parts:
        s = RefSession(ref, [pieces[i][0] for i in part], [pieces[i][1] for i in part],
                       [pieces[i][2] for i in part], cfg)
        s.wrap([pieces[i][3] for i in part])
        sessions.append(s)
    with ThreadPoolExecutor(max_workers=len(sessions)) as ex:
        for _ in range(warm):
            list(ex.map(lambda s: s.step_wrapped(), sessions))
        t0 = time.perf_counter()
        for _ in range(reps):
            list(ex.map(lambda s: s.step_wrapped(), sessions))
        dt = (time.perf_counter() - t0) / reps
    for s in sessions:
        s.close()
    return {"sec": dt, "threads": len(sessions), "balance": balance, "pieces": len(pieces)}


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_sample_layers(wl, nb: int, wte_rows: int):
    """The bounded CPU sample of a GPT workload: the first `nb` transformer
    blocks plus the first `wte_rows` rows of the token embedding.  Returns
    [(tensor index, dense offset, dense length)]."""
    blocks = gpt_blocks_of(wl)
    sel = [(i, 0, wl.tensors[i].numel) for b in blocks[:nb] for i in b]
    names = [t.name for t in wl.tensors]
    if wte_rows and "wte" in names:
        i = names.index("wte")
        sel.append((i, 0, min(wte_rows, wl.tensors[i].shape[0]) * wl.tensors[i].shape[1]))
    return sel, len(blocks)


def cpu_baseline_pair(dense_len, idx_sets, theta_sets, grad_sets, cfg_vals, reps, reps1):
    """Both CPU baselines on one sample: the reference as shipped (1 thread)
    and on every usable host thread with balanced element ranges."""
    one = cpu_reference_sample(dense_len, idx_sets, theta_sets, grad_sets, cfg_vals, reps=reps1,
                               warm=1, threads=1)
    allt = cpu_reference_sample(dense_len, idx_sets, theta_sets, grad_sets, cfg_vals, reps=reps,
                                warm=1)
    return one, allt


# ---------------------------------------------------------------------------
# reference arm

def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np

    from oracle.oracle import Oracle, RefLib, build
    from paper_2302_05045_b200 import workloads
    build()
    wl = workloads.get(args.workload, args.sparsity)
    o = Oracle()
    ref = RefLib()
    ncores = len(os.sched_getaffinity(0))
    nb = args.cpu_blocks or (2 if ncores >= 8 else 1)
    sel, nblocks = cpu_sample_layers(wl, nb, args.cpu_wte_rows)
    dense_len = [n for _, _, n in sel]
    # inputs: the same counter-hash synthetic values as the GPU arm (the
    # embedding rows are the first rows of the GPU arm's wte)
    vals = [o.synth_f32(off, n, args.seed, 2 * i, wl.tensors[i].init_bound) for i, off, n in sel]
    from concurrent.futures import ThreadPoolExecutor

    def prune_one(j):  # the reference's own magnitude_prune, per layer
        rc, s = ref.magnitude_prune([vals[j]], [wl.tensors[sel[j][0]].prunable], wl.sparsity, 0)
        assert rc == 0
        return s[0]
    with ThreadPoolExecutor(max_workers=ncores) as ex:
        idx = list(ex.map(prune_one, range(len(sel))))
    theta = [o.compress(v, s) for v, s in zip(vals, idx)]
    grads = [o.synth_f16(off, n, args.seed + 1, 2 * i + 1, 2.0**-7, 1024.0) for i, off, n in sel]
    del vals
    phi_s = sum(dense_len)
    cfg = (1e-3, 0.9, 0.999, 1e-8, 1024.0, 0.0)
    steps = max(1, args.steps)
    one, allt = cpu_baseline_pair(dense_len, idx, theta, grads, cfg, reps=steps, reps1=1)
    dt = allt["sec"]
    value = phi_s / dt
    sample = (f"{nb} of {nblocks} transformer blocks of {wl.name} + the first {args.cpu_wte_rows} "
              f"rows of wte (masked on their own) = {len(sel)} tensors, {phi_s} params per step; "
              f"sink gather + SamoTrainer::optimizer_step of the unmodified reference, cut into "
              f"{allt['pieces']} element ranges over {allt['threads']} independent trainers "
              f"(max/mean thread load {allt['balance']:.3f})")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "ms_per_step_extrapolated": dt * 1e3 * wl.phi / phi_s,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": {"workload": wl.name, "sparsity": wl.sparsity,
                                        "phi": wl.phi, "sample_params": phi_s,
                                        "parallelism": "cpu-threads"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": allt["threads"], "kind": "reference",
                         "sample": sample, "load_balance": allt["balance"], "cpu": cpu_model(),
                         "single_thread": {"value": phi_s / one["sec"], "unit": UNIT,
                                           "ms_per_step": one["sec"] * 1e3,
                                           "note": "the reference as shipped: one trainer, "
                                                   "layers whole (train.hpp:617-656)"}},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "ms_per_step is the measured sample step; ms_per_step_extrapolated scales it to "
                "the whole workload (phi / sample params)",
    }
    emit(line)


# ---------------------------------------------------------------------------
# SAMO arm

def fused_sink_probe(reps: int = 10) -> dict:
    """SURVEY §8(f)-1 (not the headline): one GPT-2.7B MLP layer (4096 tokens,
    2560 x 10240, p = 0.9) — the weight-gradient GEMM with the gather fused
    into its epilogue (samo_model_sink_dw) vs the dense GEMM + K1 on the layer,
    and cuBLAS for the GEMM alone.  CUDA events around `reps` back-to-back
    calls, best of 3."""
    import torch
    from paper_2302_05045_b200 import samo
    batch, n_in, n_out, p = 4096, 2560, 10240, 0.9
    g = torch.Generator(device="cuda").manual_seed(1)
    x = (torch.rand(batch, n_in, device="cuda", generator=g) * 2 - 1).half()
    dy = ((torch.rand(batch, n_out, device="cuda", generator=g) * 2 - 1) * 4).half()
    n = n_in * n_out
    idx = torch.randperm(n, device="cuda", generator=g)[: int(round((1 - p) * n))].sort().values.to(torch.int32)
    m = samo.SamoModel.from_index_sets([samo.PrunedIndexSet("mlp.fc_in.weight", n, idx)], [(n_in, n_out)], 0)
    m.init_layer(0, torch.zeros(n, device="cuda"))

    def timed(fn):  # back-to-back calls between two events, best of 3
        for _ in range(3):
            fn()
        best = float("inf")
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                fn()
            b.record()
            b.synchronize()
            best = min(best, a.elapsed_time(b) / reps)
        return best

    flops = 2.0 * batch * n_in * n_out
    t_gemm = timed(lambda: samo.dw_gemm(x, dy))
    t_cublas = timed(lambda: torch.matmul(x.t(), dy))
    t_unfused = timed(lambda: m.sink_dense(0, samo.dw_gemm(x, dy).reshape(-1)))
    t_fused = timed(lambda: m.sink_dw(0, x, dy))
    m._sink_keepalive.clear()
    m.close()
    pk = peaks()
    return {"shape": {"batch": batch, "in": n_in, "out": n_out, "sparsity": p},
            "dw_gemm_ms": t_gemm, "dw_gemm_tflops": flops / t_gemm / 1e9,
            "roofline": {"bound": "tensor", "achieved": flops / t_gemm / 1e9, "peak": pk.get("bf16_tflops"),
                         "unit": "TFLOP/s",
                         "frac": (flops / t_gemm / 1e9) / pk["bf16_tflops"] if pk.get("bf16_tflops") else None},
            "cublas_ms": t_cublas, "cublas_tflops": flops / t_cublas / 1e9,
            "unfused_sink_ms": t_unfused, "fused_sink_ms": t_fused,
            "fused_saving": 1 - t_fused / t_unfused}


def mix_ceiling(k: dict):
    """The measured streaming ceiling of the HBM read:write mix nearest to
    the kernel's own (tools/bw_probe.cu on B200, profiles/r02l_bw_probe.jsonl):
    register streams (LDG/STG) of each mix, and for the 1:1 mix also a copy
    through the TMA engines, whichever is higher — the step kernels stage
    their reads with TMA, and the TMA copy is the fastest copy measured on
    this box (6724 GB/s, above the driver's torch-copy figure).  Reported
    beside `frac`, never instead of it."""
    if "write_bytes" not in k:
        return None
    try:
        pts = [json.loads(l) for l in (ROOT / "profiles" / "r02l_bw_probe.jsonl").read_text().splitlines()
               if l.strip()]
    except OSError:
        return None
    reg = [p for p in pts if "read_streams" in p]
    w = k["write_bytes"] / k["bytes"]
    best = min(reg, key=lambda p: abs(p["write_streams"] / (p["read_streams"] + p["write_streams"]) - w))
    gbps, mix = best["GBps"], best["mix"]
    if best["read_streams"] == best["write_streams"]:
        tma = [p["GBps"] for p in pts if p.get("mix") == "tma copy 1:1"]
        if tma and max(tma) > gbps:
            gbps, mix = max(tma), "copy 1:1 through TMA (cp.async.bulk both ways)"
    return {"mix": mix, "write_fraction": round(w, 3), "GBps": gbps,
            "frac": k["GBps"] / gbps, "src": "tools/bw_probe.cu"}


class gpu_local_cpus:
    """Runs the block bound to the CPUs NVML reports as local to `dev`
    (nvmlDeviceGetCpuAffinity), then restores the affinity.  A pinned host
    buffer allocated inside is placed on the GPU's NUMA node, so its
    host->device copies do not cross the socket interconnect.  No-op where
    NVML or the mapping is unavailable, or with SAMO_BENCH_NUMA=0."""

    def __init__(self, dev):
        self.dev, self.saved = dev, None

    def __enter__(self):
        if os.environ.get("SAMO_BENCH_NUMA", "1") == "0" or not hasattr(os, "sched_setaffinity"):
            return self
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            uuid = str(torch.cuda.get_device_properties(self.dev).uuid)
            h = pynvml.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
            words = pynvml.nvmlDeviceGetCpuAffinity(h, 64)
            cpus = {64 * w + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}
            cpus &= os.sched_getaffinity(0)
            if cpus:
                self.saved = os.sched_getaffinity(0)
                os.sched_setaffinity(0, cpus)
        except Exception:  # noqa: BLE001  (no NVML / no mapping: leave placement to the OS)
            self.saved = None
        return self

    def __exit__(self, *exc):
        if self.saved:
            os.sched_setaffinity(0, self.saved)
        return False


def fc_sweep_probe(reps: int = 200, cpu: bool = True) -> list:
    """BASELINE config 2 (config 1 = its 4096 row): one [n, n]
    FC layer, 90% magnitude mask (K0), loss-scaled binary16 gradients.  The
    device step as a CUDA graph — L2-resident, so this is latency, reported
    per step — next to the reference's own step (oracle/_ref: sink gather +
    SamoTrainer::optimizer_step, single thread as shipped) on the same data."""
    import numpy as np
    import torch

    from paper_2302_05045_b200 import samo, workloads
    ref_reps = {128: 1000, 256: 300, 512: 100, 1024: 30, 2048: 10, 4096: 3}
    out = []
    for n in (128, 256, 512, 1024, 2048, 4096):
        wl = workloads.fc(n, 0.9)
        t = wl.tensors[0]
        w = samo.synth_uniform_f32(t.numel, 7, 0, t.init_bound)
        sets = samo.magnitude_prune([samo.LayerParams(t.name, w, True)], 0.9)
        m = samo.SamoModel.from_index_sets(sets, [t.shape])
        m.init_layer(0, w)
        m.set_config(samo.OptimizerConfig())
        theta0 = m.read(0, "theta32").cpu().numpy()
        g = samo.synth_uniform_f16(t.numel, 8, 1, 2.0**-7, 1024.0)
        m.set_grads([g])
        for _ in range(10):
            m.step(graph=True)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            m.step(graph=True)
        b.record()
        b.synchronize()
        us = a.elapsed_time(b) * 1000.0 / reps
        entry = {"workload": wl.name, "params": t.numel, "kept": int(sets[0].count()),
                 "step_us": us, "params_per_s": t.numel / (us * 1e-6)}
        if cpu:
            try:
                idx = sets[0].indices.cpu().numpy().view(np.uint32)
                gh = g.cpu().numpy().view(np.uint16)
                dt = cpu_reference_sample([t.numel], [idx], [theta0], [gh],
                                          (1e-3, 0.9, 0.999, 1e-8, 1024.0, 0.0), reps=ref_reps[n],
                                          threads=1)["sec"]
                entry["reference_cpu_us"] = dt * 1e6
                entry["speedup_vs_reference"] = dt * 1e6 / us
            except Exception as ex:  # no oracle/_ref on this host
                entry["reference_cpu_us"] = None
                entry["reference_error"] = str(ex)
        m.close()
        out.append(entry)
    return out


def run_samo(args) -> None:
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2302_05045_b200 import _abi, samo, workloads
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)

    wl = workloads.get(args.workload, args.sparsity)
    L = len(wl.tensors)
    t_setup = time.perf_counter()

    # -- one-time: synthetic weights, K0 magnitude prune, model state ------
    sets, shapes = [], []
    init_vals = []
    for i, t in enumerate(wl.tensors):
        v = samo.synth_uniform_f32(t.numel, args.seed, 2 * i, t.init_bound)
        init_vals.append(v)
        shapes.append(t.shape)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    sets = samo.magnitude_prune([samo.LayerParams(t.name, v, t.prunable)
                                 for t, v in zip(wl.tensors, init_vals)], wl.sparsity)
    ev1.record()
    torch.cuda.synchronize()
    prune_ms = ev0.elapsed_time(ev1)
    model = samo.SamoModel.from_index_sets(sets, shapes, args.tile)
    for l, v in enumerate(init_vals):
        model.init_layer(l, v)
    cfg = samo.OptimizerConfig()
    model.set_config(cfg)
    phi, nnz, ntiles = model.totals()
    torch.cuda.synchronize()
    cpu_sample = None
    # (the reference is binary16-only: no CPU baseline for bf16 gradients)
    if rank == 0 and world == 1 and not (args.no_cpu_baseline or args.profile or args.grad_dtype == "bf16"):
        # keep what the CPU sample needs (the K0 masks, bit-exact with the
        # reference's) before freeing the dense init values
        ncores = len(os.sched_getaffinity(0))
        nb = args.cpu_blocks or (2 if ncores >= 8 else 1)
        sel, nblocks = cpu_sample_layers(wl, nb, args.cpu_wte_rows)
        cs_idx, cs_theta = [], []
        for i, off, n in sel:
            idx = sets[i].indices.cpu().numpy().view(np.uint32)
            th = model.read(i, "theta32").cpu().numpy()
            a, b = np.searchsorted(idx, off), np.searchsorted(idx, off + n)
            cs_idx.append((idx[a:b] - np.uint32(off)).astype(np.uint32))
            cs_theta.append(th[a:b].copy())
        cpu_sample = {"sel": sel, "nb": nb, "nblocks": nblocks, "idx": cs_idx, "theta": cs_theta}
    # 32-byte theta16 sectors (16 values) holding a kept element: the sectors
    # K123 writes (the others stay zero)
    sectors16 = int(sum(int(torch.unique_consecutive(st.as_int64() >> 4).numel()) if st.count() else 0
                        for st in sets))
    del init_vals, sets
    torch.cuda.empty_cache()

    # -- dense binary16 gradients: one flat arena, 256-byte aligned segments --
    offs, off = [], 0
    for t in wl.tensors:
        offs.append(off)
        off += (t.numel + 127) // 128 * 128
    grad_arena = torch.empty(off, dtype=torch.float16, device=dev)
    grads = []
    for i, t in enumerate(wl.tensors):
        g = grad_arena[offs[i]:offs[i] + t.numel]
        samo.synth_uniform_f16(t.numel, args.seed + 1 + rank, 2 * i + 1, 2.0**-7, 1024.0, out=g)  # rank_seed
        grads.append(g)
    if args.grad_dtype == "bf16":  # the same values rounded to bfloat16 (setup, untimed)
        grad_arena = grad_arena.float().to(torch.bfloat16)
        grads = [grad_arena[offs[i]:offs[i] + t.numel] for i, t in enumerate(wl.tensors)]
        model.set_grad_dtype(torch.bfloat16)
    model.set_grads(grads)

    comm = None
    if world > 1:
        from paper_2302_05045_b200 import dist as sdist
        comm = sdist.make_communicator()
        model.attach_comm(comm)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup

    # -- warm-up (graph path: also validates the captured step) --------------
    for _ in range(max(0, args.warmup)):
        model.step(graph=True)
    torch.cuda.synchronize()

    # -- timed region: staged step with events between the stages -----------
    K = max(1, args.steps)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K)]
    gpu_name = torch.cuda.get_device_properties(dev).name
    smi_index = os.environ.get("CUDA_VISIBLE_DEVICES", str(local)).split(",")[local] \
        if os.environ.get("CUDA_VISIBLE_DEVICES") else str(local)
    # The same K steps timed once without any clock sampling first: every NVML
    # clock query stalls the GPU for a few ms (ClockSampler), which the timed
    # region below pays; this figure shows by how much (diagnostic only).
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    u0, u1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    u0.record()
    for s in range(K):
        model.step(graph=args.graph) if world == 1 else model.step()
    u1.record()
    torch.cuda.synchronize()
    unsampled_ms = u0.elapsed_time(u1)
    if world > 1:
        ut = torch.tensor([unsampled_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(ut, op=dist.ReduceOp.MAX)
        unsampled_ms = float(ut.item())
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = samo.kernel_launch_count()
    nvl = nvl0 = None
    if world > 1 and os.environ.get("SAMO_BENCH_NVLINK") == "1":  # NVLink bytes sent / received (NVML)
        try:
            from paper_2302_05045_b200.nvlink import NvlinkBytes
            nvl = NvlinkBytes(int(smi_index))
            nvl0 = nvl.read()
        except Exception as ex:  # noqa: BLE001  (no NVML counter: reported as unavailable)
            nvl, nvl0 = None, str(ex)
    with ClockSampler(smi_index if rank == 0 else None) as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        if world == 1:
            # the production single-GPU step: K123 (+ the skip-repair no-op),
            # eager launches or one captured graph per step
            for s in range(K):
                model.step(graph=args.graph)
        else:
            # the production data-parallel step: bucketed exchange overlapped
            # with the gather and update kernels
            for s in range(K):
                model.step()
        t1.record()
        clk.sample_now()  # the queued steps are still running
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        # keep sampling a little longer so short regions still get clock samples
        t_end = time.perf_counter() + 1.0
        while clk.active() and len(clk) < 3 and time.perf_counter() < t_end:
            time.sleep(0.05)
    launches = samo.kernel_launch_count() - launches0
    total_ms = t0.elapsed_time(t1)
    nvlink_measured = None
    if world > 1:  # every rank joins the gather (NaN where NVML has no counter)
        nvl1 = nvl.read() if nvl is not None else None
        per = torch.tensor([(nvl1[0] - nvl0[0]) / K, (nvl1[1] - nvl0[1]) / K] if nvl1 else
                           [float("nan")] * 2, device=dev, dtype=torch.float64)
        allr = [torch.zeros_like(per) for _ in range(world)]
        dist.all_gather(allr, per)
        if nvl is not None:
            nvlink_measured = {"source": f"NVML {nvl.source} counters, {len(nvl.links)} links",
                               "tx_bytes_per_step_per_rank": [float(x[0]) for x in allr],
                               "rx_bytes_per_step_per_rank": [float(x[1]) for x in allr],
                               "note": "whole device over the timed region (all kernels, NCCL "
                                       "barriers included), divided by the steps"}
        else:
            nvlink_measured = {"unavailable": nvl0 or "NVML NVLink counters not read (SAMO_BENCH_NVLINK=1 reads them)"}
    phases = pipeline = overlap = None
    fused_ms = None
    fused = world == 1 and os.environ.get("SAMO_FUSED_STEP", "1") != "0"
    KB = min(K, 10)
    if world == 1:
        # Per-kernel breakdown (not the headline): the fused step's kernels
        # timed by events inside the driver, one step at a time; then the
        # K1 | K23 pair of the split path on the same state, for comparison.
        if fused:
            fused_ms = []
            _abi.call("samo_model_enable_phase_timing", model.handle, 1)
            for _ in range(KB):
                model.step()
                buf = (C.c_float * 4)()
                cnt = _abi.load().samo_model_phase_times(model.handle, buf, 4)
                fused_ms.append([buf[i] for i in range(max(0, cnt))])
            _abi.call("samo_model_enable_phase_timing", model.handle, 0)
        evs = evs[:KB]
        for s in range(KB):
            e = evs[s]
            e[0].record()
            model.gather()
            e[1].record()
            model.exchange()  # no-op without a communicator
            e[2].record()
            model.update()
            e[3].record()
        torch.cuda.synchronize()
    if world > 1:
        tt = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
        # Phase breakdown of the production step (events inside the driver;
        # sharded exchange only) — not the headline.
        phases = None
        pipeline = None
        overlap = None

        def phase_pass():
            _abi.call("samo_model_enable_phase_timing", model.handle, 1)
            for _ in range(3):
                model.step()
            buf = (C.c_float * 16)()
            cnt = _abi.load().samo_model_phase_times(model.handle, buf, 16)
            _abi.call("samo_model_enable_phase_timing", model.handle, 0)
            return [round(buf[i], 4) for i in range(max(0, cnt))]

        if model.exchange_mode() == model.EXCHANGE_P2P:
            ph = phase_pass()
            if len(ph) == 4:  # pipelined step (SAMO_P2P_BUCKETS > 1)
                pipeline = dict(zip(["K1_gather", "skip-flag exchange (peer signals)",
                                     "shard update || expand (pipelined over k-buckets)",
                                     "finalize"], ph))
                # per-kernel breakdown from the serial schedule of the same kernels
                old_b = os.environ.get("SAMO_P2P_BUCKETS")
                os.environ["SAMO_P2P_BUCKETS"] = "1"
                ph = phase_pass()
                if old_b is None:
                    del os.environ["SAMO_P2P_BUCKETS"]
                else:
                    os.environ["SAMO_P2P_BUCKETS"] = old_b
            phases = dict(zip(["K1_gather", "skip-flag allreduce (barrier)",
                               "shard update: fused NVLink exchange + Adam", "norm allreduce (barrier)",
                               "expand", "finalize"], ph))
            overlap = sunk_pass(model, grads, stream, dev)
        elif model.exchange_mode() == model.EXCHANGE_SHARDED:
            phases = dict(zip(["K1_gather (reduce-scatter overlapped)",
                               "skip flag + shard Adam + first all-gather bucket",
                               "expand (all-gather overlapped)", "norm allreduce + finalize"], phase_pass()))
        # Stage breakdown (not the headline): the same three stages run back
        # to back, the exchange as one allreduce of the whole arena.
        KB = min(K, 10)
        evs = evs[:KB]
        dist.barrier()
        torch.cuda.synchronize()
        for s in range(KB):
            e = evs[s]
            e[0].record()
            model.gather()
            e[1].record()
            model.exchange()
            e[2].record()
            model.update()
            e[3].record()
        torch.cuda.synchronize()
    k1 = [e[0].elapsed_time(e[1]) for e in evs]
    ar = [e[1].elapsed_time(e[2]) for e in evs]
    k23 = [e[2].elapsed_time(e[3]) for e in evs]
    ms_step = total_ms / K
    rec = model.step_record()
    value = world * phi / (ms_step * 1e-3)

    pk = peaks()
    p2p = world > 1 and model.exchange_mode() == model.EXCHANGE_P2P and phases
    k1_ms = statistics.mean(k1)
    k23_ms = statistics.mean(k23)
    ar_ms = statistics.mean(ar)
    if not p2p:
        # Algorithmic bytes per launch: dense grad read 2phi +
        # off16 2n + compressed grad write (fp32 4n when exchanged, binary16 2n
        # otherwise); K23: grad read + off16 2n + theta/m/v read+write 24n +
        # dense theta16 write 2phi.
        gb = 4 if world > 1 else 2
        bytes_k1 = 2 * phi + 2 * nnz + gb * nnz
        bytes_k23 = 2 * phi + 2 * nnz + gb * nnz + 24 * nnz
        kern = {
            "K1_gather_unscale": {"ms": k1_ms, "bytes": bytes_k1,
                                  "GBps": bytes_k1 / (k1_ms * 1e-3) / 1e9,
                                  "write_bytes": gb * nnz},
            "K23_adam_downcast_expand": {"ms": k23_ms, "bytes": bytes_k23,
                                         "GBps": bytes_k23 / (k23_ms * 1e-3) / 1e9,
                                         "write_bytes": 12 * nnz + 2 * phi},
        }
        hbm_kernels = list(kern)
        if fused:
            # K123: dense grad 2phi + off16 2n + theta/m/v read
            # 12n + theta/m/v write 12n + the theta16 sectors holding a kept
            # element (32 B each), one launch per step.
            for v in kern.values():
                v["role"] = "split path (SAMO_FUSED_STEP=0), timed for comparison"
            f_ms = statistics.mean(x[0] for x in fused_ms)
            r_ms = statistics.mean(x[1] for x in fused_ms)
            b_f = 2 * phi + 26 * nnz + 32 * sectors16
            kern["K123_fused_step"] = {"ms": f_ms, "bytes": b_f, "GBps": b_f / (f_ms * 1e-3) / 1e9,
                                       "write_bytes": 32 * sectors16 + 12 * nnz,
                                       "theta16_sectors_written": sectors16,
                                       "theta16_sector_fraction": 32 * sectors16 / (2 * phi)}
            kern["k123_repair"] = {"ms": r_ms, "bytes": 0, "GBps": 0.0,
                                   "note": "skip repair: returns at once unless the step was skipped"}
            hbm_kernels = ["K123_fused_step"]
            bytes_k1, bytes_k23, k1_ms, k23_ms = 0, b_f, 0.0, f_ms
    else:
        # Production data-parallel step (fused P2P exchange), per rank
        # (DESIGN.md §7), push mode (default): K1 2phi + 2n off16 + 2n grad16,
        # the grad16 of other owners' shards going out over NVLink
        # (2n(G-1)/G per direction); shard update: the G contributions to the
        # own shard from the local receive buffer (2n) + own theta/m/v r+w
        # 24n/G + every owner storing binary16 weights here (2n), binary16
        # weights out over NVLink 2n(G-1)/G per direction; expand 2n
        # theta16c + 2n off16 + 2phi.  Pull mode (SAMO_P2P_PUSH=0): the shard
        # kernel also loads the other ranks' grad16 over NVLink.
        G = world
        push = os.environ.get("SAMO_P2P_PUSH", "1") != "0"
        ph = list(phases.values())
        sh_ms, ex_ms = ph[2], ph[4]
        k1_ms = ph[0]
        b_k1 = 2 * phi + 4 * nnz
        b_sh = 24 * nnz // G + 4 * nnz
        b_nv = (2 if push else 4) * nnz * (G - 1) // G
        b_ex = 2 * phi + 4 * nnz
        kern = {
            "K1_gather": {"ms": k1_ms, "bytes": b_k1, "GBps": b_k1 / (k1_ms * 1e-3) / 1e9,
                          "nvlink_bytes_per_direction": (2 * nnz * (G - 1) // G) if push else 0},
            "shard_update_p2p": {"ms": sh_ms, "bytes": b_sh, "GBps": b_sh / (sh_ms * 1e-3) / 1e9,
                                 "nvlink_bytes_per_direction": b_nv,
                                 "nvlink_GBps_per_direction": b_nv / (sh_ms * 1e-3) / 1e9,
                                 "nvlink_frac_of_900": b_nv / (sh_ms * 1e-3) / 900e9},
            "expand": {"ms": ex_ms, "bytes": b_ex, "GBps": b_ex / (ex_ms * 1e-3) / 1e9},
        }
        hbm_kernels = ["K1_gather", "expand"]
        bytes_k1, bytes_k23 = b_k1, b_sh + b_ex
        k23_ms = sh_ms + ex_ms
    for v in kern.values():
        v["frac"] = v["GBps"] / pk["hbm_gbs"]
    if world > 1:
        msg = 4 * (nnz + 1)
        kern["nccl_allreduce_reference"] = {
            "ms": ar_ms, "bytes": msg, "algbw_GBps": msg / (ar_ms * 1e-3) / 1e9,
            "note": "standalone NCCL allreduce of the whole compressed fp32 arena (the "
                    "replicated-exchange alternative), for context",
            "busbw_GBps": msg * 2 * (world - 1) / world / (ar_ms * 1e-3) / 1e9,
            "busbw_frac_of_900": msg * 2 * (world - 1) / world / (ar_ms * 1e-3) / 900e9}
    dom = max(hbm_kernels, key=lambda k: kern[k]["ms"])
    traffic = None
    tp = ROOT / "profiles" / "traffic.json"
    if tp.exists() and not p2p:
        try:
            traffic = json.loads(tp.read_text()).get(wl.name, {}).get(dom)
        except (ValueError, AttributeError):
            traffic = None
    mix = mix_ceiling(kern[dom])
    roofline = {"bound": "hbm", "kernel": dom, "achieved": kern[dom]["GBps"], "peak": pk["hbm_gbs"],
                "mix_ceiling": mix,
                "nominal": {"GBps": 8000.0, "frac": kern[dom]["GBps"] / 8000.0,
                            "note": "B200 HBM3e data-sheet bandwidth; the measured peaks sit below it"},
                "peak_src": pk["src"], "unit": "GB/s", "frac": kern[dom]["frac"], "traffic": traffic,
                "algorithmic_bytes_per_launch": kern[dom]["bytes"],
                "step_bytes": bytes_k1 + bytes_k23,
                "step_frac": (bytes_k1 + bytes_k23) / ((k1_ms + k23_ms) * 1e-3) / 1e9 / pk["hbm_gbs"]}

    # -- e2e: public API with HOST buffers (pinned), copies inside the region --
    e2e = None
    e2e_ok = not (args.no_e2e or args.profile)
    if e2e_ok:
        # The pinned staging buffer (5.3 GB per rank) is the one allocation
        # that can fail on a small host; every rank agrees before going on.
        try:
            with gpu_local_cpus(dev):  # pages placed on the GPU's NUMA node
                host = torch.empty(off, dtype=grad_arena.dtype, pin_memory=True)
        except Exception as ex:  # noqa: BLE001
            host, e2e_err = None, str(ex)
        ok = torch.tensor([1 if host is not None else 0], device=dev, dtype=torch.int32)
        if world > 1:
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        e2e_ok = bool(ok.item())
        if not e2e_ok:
            e2e = {"value": None, "error": f"pinned host staging buffer unavailable: {e2e_err if host is None else 'on another rank'}"}
            host = None
    if e2e_ok:
        E = args.e2e_steps or min(K, 10)
        host.copy_(grad_arena)  # this rank's synthetic gradients, staged on the host
        dbuf = [grad_arena, torch.empty_like(grad_arena)]
        dgrads = [[d[offs[i]:offs[i] + t.numel] for i, t in enumerate(wl.tensors)] for d in dbuf]
        rec_host = torch.empty(32, dtype=torch.uint8, pin_memory=True)
        copy_stream = torch.cuda.Stream(device=dev)
        h2d_done = [torch.cuda.Event() for _ in range(2)]
        consumed = [torch.cuda.Event() for _ in range(2)]
        for c in consumed:
            c.record(stream)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(stream)

        def h2d(s):
            b = s % 2
            with torch.cuda.stream(copy_stream):
                copy_stream.wait_event(consumed[b])
                dbuf[b].copy_(host, non_blocking=True)
                h2d_done[b].record(copy_stream)
        h2d(0)
        for s in range(E):
            if s + 1 < E:
                h2d(s + 1)
            b = s % 2
            stream.wait_event(h2d_done[b])
            model.set_grads(dgrads[b])
            model.step()  # the production step (P2P exchange at N > 1)
            consumed[b].record(stream)
            _abi.call("samo_model_step_record_async", model.handle, C.c_void_p(rec_host.data_ptr()),
                      C.c_void_p(stream.cuda_stream))
        a1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = a0.elapsed_time(a1)
        if world > 1:
            tt = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_ms = float(tt.item())
        e2e = {"value": world * phi / (e2e_ms / E * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(host.numel() * 2), "d2h_bytes_per_step": 32,
               "steps": E, "ms_per_step": e2e_ms / E,
               "note": f"dense {args.grad_dtype} grads H2D from pinned host (double-buffered against the "
                       "previous step; PCIe-bound: 55.5 GB/s with 1-8 copy streams, "
                       "tools/h2d_probe.py) + step + D2H of the step record (grad norm, skip flag)"}
        del host, dbuf, dgrads

    # -- CPU baseline: the reference on this host, bounded sample ------------
    cpu = None
    if cpu_sample is not None:
        sel = cpu_sample["sel"]
        dl = [n for _, _, n in sel]
        gr = [grads[i][off:off + n].cpu().numpy().view(np.uint16) for i, off, n in sel]
        cfgv = (cfg.learning_rate, cfg.beta1, cfg.beta2, cfg.epsilon, cfg.loss_scale, cfg.weight_decay)
        try:
            one, allt = cpu_baseline_pair(dl, cpu_sample["idx"], cpu_sample["theta"], gr, cfgv,
                                          reps=3, reps1=1)
            phi_s = sum(dl)
            cpu = {"value": phi_s / allt["sec"], "unit": UNIT, "cores": allt["threads"], "kind": "reference",
                   "sample": f"{cpu_sample['nb']} of {cpu_sample['nblocks']} transformer blocks + the "
                             f"first {args.cpu_wte_rows} rows of wte ({len(sel)} tensors, {phi_s} params), "
                             f"sink gather + SamoTrainer::optimizer_step of the unmodified reference, "
                             f"cut into {allt['pieces']} element ranges over {allt['threads']} "
                             f"independent trainers, 3 reps",
                   "load_balance": allt["balance"], "cpu": cpu_model(), "ms_per_sample_step": allt["sec"] * 1e3,
                   "single_thread": {"value": phi_s / one["sec"], "unit": UNIT,
                                     "ms_per_sample_step": one["sec"] * 1e3,
                                     "note": "the reference as shipped: one trainer, layers whole"}}
        except Exception as ex:  # the baseline must not kill the GPU measurement
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                   "sample": f"failed: {ex}"}

    fused = fc_sweep = None
    if world == 1 and not (args.profile or args.no_fused):
        try:
            fused = fused_sink_probe()
        except Exception as ex:  # a probe failure must not drop the headline line
            fused = {"error": str(ex)}
        try:
            fc_sweep = fc_sweep_probe(cpu=not args.no_cpu_baseline)
        except Exception as ex:
            fc_sweep = [{"error": str(ex)}]

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": f"synthetic (counter-hash weights and loss-scaled {'bf16' if args.grad_dtype == 'bf16' else 'fp16'} "
                    "grads; K0-pruned mask)",
            "config": {"workload": wl.name, "description": wl.description,
                       "sparsity": wl.sparsity, "phi": phi, "nnz": nnz, "tensors": L,
                       "tiles": ntiles, "parallelism": f"dp{world}", "grad_dtype": args.grad_dtype,
                       "l2": (f"inputs ({(4 * phi + 32 * nnz) / 1e9:.1f} GB per step) are larger than "
                              "L2; no flush needed") if 4 * phi + 32 * nnz > 2 * 126e6 else
                             "L2-resident working set: latency-bound configuration, reported as "
                             "time per step (no flush between steps)",
                       "timing": ("CUDA graph per step" if args.graph else "eager launches") +
                                 ", CUDA events around the timed region on the launching stream",
                       "gpu": gpu_name},
            "gpu_launches": int(launches),
            "step_mode": ("K123 fused step (gather + unscale + Adam + downcast + expand, one pass per "
                          "tile, speculative on the skip flag) + skip-repair no-op" if fused else
                          "K1 | K23 (no exchange)") if world == 1 else
                         ("p2p (ZeRO-1, exchange fused over NVLink, no NCCL): K1 pushes each kept "
                          "binary16 grad into its owner's receive buffer | peer-signalled flag "
                          "exchange | per k-bucket: shard kernel sums the G local contributions "
                          "in rank order, Adam, stores binary16 weights to every rank, signals "
                          "the bucket || expand of the signalled buckets"
                          if model.exchange_mode() == model.EXCHANGE_P2P else
                          "sharded (ZeRO-1), k-bucketed: K1 || NCCL reduce-scatter, shard Adam, "
                          "NCCL all-gather of binary16 weights || expand"
                          if model.exchange_mode() == model.EXCHANGE_SHARDED
                          else "allreduce: bucketed NCCL allreduce overlapped with K1/K23"),
            "model_params_per_s": phi / (ms_step * 1e-3),
            "nvlink_measured": nvlink_measured,
            "phases_ms": phases,
            "pipeline_phases_ms": pipeline,
            "backward_overlap": overlap,
            "p2p_features": model.p2p_features() if world > 1 else None,
            "roofline": roofline,
            "kernels": kern,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "fused_dw_sink": fused,
            "fc_sweep": fc_sweep,
            "clocks": clk.summary(),
            "unsampled": {"ms_per_step": unsampled_ms / K,
                          "note": "the same steps timed just before, with no clock sampling (each NVML "
                                  "clock query stalls the GPU for a few ms; the headline keeps the sampled "
                                  "region, DESIGN §6)"},
            "step_record": {"t": int(rec.t), "skipped": int(rec.skipped_steps),
                            "grad_norm": float(rec.grad_norm)},
            "setup": {"seconds": setup_s, "k0_prune_ms": prune_ms,
                      "model_device_bytes": model.device_bytes()},
        }
        emit(line)
    model.close()
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


_RESULT_FD = None  # the process's real stdout: only the JSON line goes there


def emit(line: dict) -> None:
    """Writes the one JSON result line to the real stdout."""
    text = (json.dumps(line) + "\n").encode()
    if _RESULT_FD is None:
        sys.stdout.write(text.decode())
        sys.stdout.flush()
    else:
        os.write(_RESULT_FD, text)


def sunk_pass(model, grads, stream, dev, reps: int = 3):
    """The exchange sent during the backward (train.hpp:287-313): per-layer
    sinks, last layer first, push each layer's kept binary16 gradients to
    their owners; step_sunk is then only the flag exchange, the shard update
    and the expand.  Times both parts (max over ranks): the sinks run back to
    back here (no backward compute to hide under), so sinks_ms is what a
    backward would absorb and step_after_sinks_ms what is left after it."""
    import torch
    import torch.distributed as dist
    L = len(grads)
    e = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(reps)]
    for r in range(reps + 1):
        dist.barrier()
        torch.cuda.synchronize()
        ev = e[r - 1] if r else None
        if ev:
            ev[0].record(stream)
        for l in reversed(range(L)):
            model.sink_dense(l, grads[l])
        if ev:
            ev[1].record(stream)
        # every rank's backward (here: its sink launches) ends before the step
        # after it, as in synchronous training, so the host-launch skew of 388
        # Python calls per rank is not charged to the step
        torch.cuda.synchronize()
        dist.barrier()
        if ev:
            ev[2].record(stream)
        model.step_sunk()
        if ev:
            ev[3].record(stream)
    torch.cuda.synchronize()
    sk = statistics.median(x[0].elapsed_time(x[1]) for x in e)
    st = statistics.median(x[2].elapsed_time(x[3]) for x in e)
    t = torch.tensor([sk, st], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return {"sinks_ms": round(float(t[0]), 4), "step_after_sinks_ms": round(float(t[1]), 4),
            "layers": L, "note": "per-layer K1 push sinks (backward order) then step_sunk (flag "
                                 "exchange + shard update || expand); the sinks' NVLink traffic "
                                 "rides under the backward in training"}


def main() -> None:
    global _RESULT_FD
    args = parse_args()
    # Everything else that reaches fd 1 — NCCL's version banner, library
    # chatter — goes to stderr, so stdout carries exactly one JSON line.
    sys.stdout.flush()
    _RESULT_FD = os.dup(1)
    os.dup2(2, 1)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_samo(args)


if __name__ == "__main__":
    main()
