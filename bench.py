"""Benchmark: stray-call analysis of the C2 synthetic corpus on B200.

Metric (BASELINE.json): source GB/s scanned (+ call-graph edges/s), with the
stray-call set bit-exact vs the CPU reference (parity is pinned by tests/).
Workload: C2 = 10,000 seeded synthetic MiniCU files of ~100 KB (~1 GB), one
GPU per 10,000 files (weak scaling over ranks), mode classic, profile nvcc 12.

A step = one full analysis of the rank's corpus: lex -> parse -> symbol join
-> instantiation fixpoint -> reachability -> ordered stray-call set.
  value : corpus already resident in HBM (exs_run_device), device time (CUDA
          events on the library stream), max over ranks.
  e2e   : the public C-ABI entry exs_run with the corpus in pinned host memory
          (H2D inside) plus the D2H read of the diagnostic records.
Inputs (1 GB) exceed the 126 MB L2, so no L2 flush is needed between steps.

--impl reference: the reference algorithm on the host CPU cores (the oracle
port in oracle/exs_oracle.py, the reference being pure Python) over a bounded
sample of the same workload, multiprocessing over all cores.
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from paper_2309_03912_b200 import synth  # noqa: E402

METRIC = "source GB/s scanned + call-graph edges/s, stray-call set bit-exact vs CPU ref"
PEAKS = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
HBM_PEAK = float(PEAKS.get("hbm_gbs", 6650.0))
HBM_PEAK_SRC = "measured" if "hbm_gbs" in PEAKS else "fallback"


def _gen(args):
    seed, size = args
    return synth.gen_c2_file(seed, size).encode()


def make_corpus(n_files: int, file_bytes: int, seed0: int, procs: int):
    with mp.Pool(procs) as pool:
        blobs = pool.map(_gen, [(seed0 + i, file_bytes) for i in range(n_files)], chunksize=32)
    offs = np.zeros(n_files + 1, dtype=np.uint64)
    offs[1:] = np.cumsum([len(b) for b in blobs])
    return blobs, offs


class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region (NVML in
    process -- the same counters nvidia-smi reports, without spawning it)."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.stop_ev = threading.Event()
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            bits = {"hw_slowdown": N.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": N.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": N.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": N.nvmlClocksEventReasonSwPowerCap}
        except Exception:
            return self._run_smi()
        while not self.stop_ev.is_set():
            try:
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append([str(sm), str(mx)] +
                                    ["Active" if r & b else "Not Active" for b in bits.values()])
            except Exception:
                pass
            self.stop_ev.wait(0.1)

    def _run_smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self.stop_ev.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self.stop_ev.wait(1.0)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop_ev.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------------------
# CPU reference arm (oracle port of the reference algorithm)

def _oracle_file(blob: bytes):
    from oracle import exs_oracle as O  # the checker/baseline only
    r = O.analyze_unit(blob.decode(), "classic")
    return len(blob), O.edge_count(r), sum(1 for d in r.diagnostics if d[0] in (
        "E1001", "E1002", "W1101", "W1102", "E1101", "E1102", "E1501", "W1502"))


def cpu_reference(n_sample: int, file_bytes: int, seed0: int, cores: int):
    """Time the reference algorithm over a bounded sample on `cores` processes."""
    blobs, _ = make_corpus(n_sample, file_bytes, seed0, cores)
    t0 = time.perf_counter()
    with mp.Pool(cores) as pool:
        res = pool.map(_oracle_file, blobs, chunksize=1)
    dt = time.perf_counter() - t0
    nbytes = sum(r[0] for r in res)
    edges = sum(r[1] for r in res)
    return {"gbs": nbytes / dt / 1e9, "edges_per_s": edges / dt, "seconds": dt, "bytes": nbytes,
            "files": n_sample}


def run_reference_arm(a, rank, world):
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    # bounded sample: ~8 files per core of the same C2 shape per step (~5 s)
    n = max(cores * 8, 32)
    vals = []
    for i in range(a.warmup + a.steps):
        r = cpu_reference(n, a.file_bytes, 10_000 + i * n, cores)
        if i >= a.warmup:
            vals.append(r)
    gbs = statistics.mean(v["gbs"] for v in vals)
    eps = statistics.mean(v["edges_per_s"] for v in vals)
    ms = statistics.mean(v["seconds"] for v in vals) * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s",
        "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (seeded C2 generator, paper_2309_03912_b200/synth.py)",
        "config": {"workload": "C2 sample: ~100 KB seeded MiniCU files, classic, nvcc 12",
                   "files_per_step": n, "file_bytes": a.file_bytes},
        "edges_per_s": eps,
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "port",
                         "sample": f"{n} C2 files (~{n * a.file_bytes / 1e6:.1f} MB) per step, "
                                   f"oracle/exs_oracle.py over {cores} processes"},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm

def run_gpu_arm(a, rank, world, local):
    import torch
    from paper_2309_03912_b200 import _native

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    procs = max(1, (os.cpu_count() or 8) // max(world, 1))
    blobs, offs = make_corpus(a.files, a.file_bytes, rank * a.files, procs)
    host = torch.frombuffer(bytearray(b"".join(blobs)), dtype=torch.uint8).pin_memory()
    nbytes = host.numel()
    dev = host.to(f"cuda:{local}", non_blocking=False)
    torch.cuda.synchronize()
    cfg = np.zeros(a.files, dtype=np.uint8)  # classic, nvcc 12
    h = _native.Handle(local)

    def run_resident():
        h.run_device(dev.data_ptr(), nbytes, offs, cfg)
        return h.stats()

    def run_e2e():
        t0 = time.perf_counter()
        h.lib.exs_run(h.h, _native.C.c_void_p(host.data_ptr()), nbytes, _native._ptr(offs),
                      a.files, _native._ptr(cfg))
        recs = h.diags(copy=False)  # D2H into pinned host memory inside exs_run; zero-copy view
        return time.perf_counter() - t0, recs.nbytes

    for _ in range(a.warmup):
        st = run_resident()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    steps = []
    kern = {}  # tag -> [total ms, launches] over the timed steps (CUDA events, library stream)
    h.set_option(2, 1)
    with ClockSampler(local) as clk:
        for _ in range(a.steps):
            steps.append(run_resident())
            for ln in h.lib.exs_profile_text().decode().splitlines():
                parts = ln.split()
                if len(parts) >= 4 and not parts[0].startswith("[") and ":" not in parts[0]:
                    k = kern.setdefault(parts[0], [0.0, 0])
                    k[0] += float(parts[1])
                    k[1] += int(parts[3].lstrip("x"))
    h.set_option(2, 0)
    torch.cuda.synchronize()
    ms = [s["ms_total"] for s in steps]
    lex_ms = [s["ms_lex"] for s in steps]
    mean_ms = statistics.mean(ms)
    # e2e through the public C ABI with host buffers
    e2e_t = []
    d2h_b = 0
    run_e2e()  # warm-up of the host-buffer path (its device staging buffer), untimed
    for _ in range(max(1, min(a.steps, 3))):
        t, d2h_b = run_e2e()
        e2e_t.append(t)
    e2e_ms = statistics.mean(e2e_t) * 1e3
    if dist:
        tt = torch.tensor([mean_ms, e2e_ms], device=f"cuda:{local}")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        mean_ms, e2e_ms = tt.tolist()
    st = steps[-1]
    total_bytes = nbytes * world
    total_edges = st["callsites"] * world
    value = total_bytes / (mean_ms / 1e3) / 1e9
    e2e = total_bytes / (e2e_ms / 1e3) / 1e9
    # roofline: the lexing stage (K1-K3): source read once + token records written
    lex_bytes = nbytes + 32 * st["tokens"]
    lex_ach = lex_bytes / (statistics.mean(lex_ms) / 1e3) / 1e9
    # per-kernel algorithmic bytes: per step
    words = nbytes // 32 + 1
    algo = {
        "lex_splice": nbytes + 4 * words,                    # source read + splice bitmap
        "lex_words": nbytes + 16 * words + words,            # source read + WScan record + flag
        "lex_count": nbytes + 4 * words,                     # source read + per-word count
        "lex_emit": nbytes + 32 * st["tokens"],              # source read + token records
        "walk_chunks": 48 * st["callsites"],                 # 48 B per edge
        "walk_roots": 48 * st["functions"],
        "parse_items": 32 * st["tokens"] + 24 * st["tokens"] // 2,
    }
    per_kernel = {}
    for tag, (ms_tot, n) in kern.items():
        ms_step = ms_tot / max(1, a.steps)
        ent = {"ms_per_step": ms_step, "launches_per_step": n / max(1, a.steps),
               "share": ms_step / mean_ms}
        if tag in algo and ms_step > 0:
            ent["achieved_gbs"] = algo[tag] / (ms_step / 1e3) / 1e9
            ent["frac"] = ent["achieved_gbs"] / HBM_PEAK
        per_kernel[tag] = ent
    dom = max(per_kernel, key=lambda k: per_kernel[k]["ms_per_step"]) if per_kernel else None
    traffic_db = {}
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if tf.exists():
        traffic_db = json.loads(tf.read_text())
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": mean_ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (seeded C2 generator, paper_2309_03912_b200/synth.py; all files distinct)",
        "config": {"workload": "C2: 10k seeded MiniCU files x ~100 KB (~1 GB) per GPU, classic, nvcc 12",
                   "files_per_gpu": a.files, "bytes_per_gpu": nbytes, "parallelism": f"dp{world} (file shards)",
                   "l2": "inputs (1 GB) larger than L2; no flush"},
        "edges_per_s": total_edges / (mean_ms / 1e3),
        "stats": {k: st[k] for k in ("tokens", "items", "functions", "instances", "callsites", "levels",
                                     "diagnostics", "retries")},
        "stage_ms": {k: statistics.mean(s[k] for s in steps) for k in ("ms_lex", "ms_parse", "ms_sema", "ms_walk")},
        "gpu_launches": int(sum(s["gpu_launches"] for s in steps)),
        # achieved = algorithmic bytes of one launch / its mean launch time (CUDA
        # events on the launching stream); traffic = measured DRAM bytes of one
        # launch (ncu dram__bytes_{read,write}.sum, profiles/ncu_traffic.json)
        "roofline": ({"bound": "hbm", "achieved": per_kernel[dom].get("achieved_gbs"),
                      "peak": HBM_PEAK, "unit": "GB/s", "frac": per_kernel[dom].get("frac"),
                      "traffic": traffic_db.get(dom, {}).get("dram_bytes_per_launch"),
                      "algorithmic_bytes": (algo[dom] / max(1.0, per_kernel[dom]["launches_per_step"])
                                            if dom in algo else None),
                      "kernel": dom, "launches_per_step": per_kernel[dom]["launches_per_step"],
                      "share_of_step": per_kernel[dom]["share"], "peak_source": HBM_PEAK_SRC,
                      "traffic_source": traffic_db.get(dom, {}).get("source")}
                     if dom else None),
        "roofline_lex_stage": {"bound": "hbm", "achieved": lex_ach, "peak": HBM_PEAK, "unit": "GB/s",
                               "frac": lex_ach / HBM_PEAK, "kernel": "lex stage K1-K3 (all launches)"},
        "kernels": per_kernel,
        "e2e": {"value": e2e, "unit": "GB/s", "h2d_bytes_per_step": int(nbytes),
                "d2h_bytes_per_step": int(d2h_b)},
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cores = os.cpu_count() or 1
        r = cpu_reference(max(cores * 16, 64), a.file_bytes, 50_000, cores)
        line["cpu_baseline"] = {"value": r["gbs"], "unit": "GB/s", "cores": cores, "kind": "port",
                                "sample": f"{r['files']} C2 files ({r['bytes'] / 1e6:.1f} MB), "
                                          f"oracle/exs_oracle.py on {cores} processes, {r['seconds']:.1f} s"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--files", type=int, default=10_000)
    ap.add_argument("--file-bytes", type=int, default=100_000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    a = ap.parse_args()
    rank, world, local = dist_env()
    if a.impl == "reference":
        run_reference_arm(a, rank, world)
    else:
        run_gpu_arm(a, rank, world, local)


if __name__ == "__main__":
    main()
