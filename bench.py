"""Benchmark: stray-call analysis of synthetic CUDA corpora on B200.

Metric (BASELINE.json): source GB/s scanned (+ call-graph edges/s), with the
stray-call set bit-exact vs the CPU reference.  Default workload C2: 10,000
seeded synthetic MiniCU files of ~100 KB (~1 GB) per GPU (weak scaling over
ranks), mode classic, profile nvcc 12.  Other BASELINE.json configs:
``--config c3`` (one unit of depth-64 template chains, ~1M instantiations per
walk), ``--config c4`` (one unit, 10M functions / 100M call edges),
``--config c5`` (lexer-stressor corpus: 8 GB per GPU, i.e. 64 GB on 8 GPUs,
streamed through the public API in batches).

A step = one full analysis of the rank's corpus: lex -> parse -> symbol join
-> instantiation fixpoint -> reachability -> verdicts -> rendered, ordered,
de-duplicated diagnostics (the reference's ``finish_diagnostics`` output).
  value : corpus already resident in HBM (exs_run_device), device time (CUDA
          events on the library stream), max over ranks.
  e2e   : the public Python API ``analyze_corpus(units)`` with the units as
          host ``str`` objects: pack into page-locked memory, H2D, analysis,
          message rendering, D2H of the results and the per-unit Analysis
          objects, wall time, max over ranks.
  parity: the oracle (CPU restatement of the reference, test infrastructure)
          on a sample of the files timed, compared with the e2e run's output.
Inputs (>= 1 GB) exceed the 126 MB L2, so no L2 flush is needed between steps.

--impl reference: the reference package itself (pip-installed unmodified into
baseline/_ref from /root/reference; pure Python) timed on the host cores over a
bounded sample of the same files, multiprocessing over all cores.

--gpus N without torchrun re-launches itself under torch.distributed.run.
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
REF_DIR = ROOT / "baseline" / "_ref"
STRAY = ("E1001", "E1002", "W1101", "W1102", "E1101", "E1102", "E1501", "W1502")


# ---------------------------------------------------------------------------
# workloads

def _gen(args):
    kind, seed, size = args
    if kind == "c5":
        return synth.gen_c5_file(seed, size, 0.01)
    return synth.gen_c2_file(seed, size)


def make_texts(kind: str, seeds, file_bytes: int, procs: int):
    with mp.Pool(procs) as pool:
        return pool.map(_gen, [(kind, s, file_bytes) for s in seeds], chunksize=16)


def make_corpus(n_files: int, file_bytes: int, seed0: int, procs: int):
    """(blobs, uint64 offsets) of C2 files seed0 .. seed0 + n_files - 1 (dev tools)."""
    blobs = [t.encode() for t in make_texts("c2", range(seed0, seed0 + n_files), file_bytes, procs)]
    offs = np.zeros(n_files + 1, dtype=np.uint64)
    offs[1:] = np.cumsum([len(b) for b in blobs])
    return blobs, offs


class Workload:
    """Units of one rank: (paths, texts) plus how to describe them."""

    def __init__(self, a, rank: int, world: int):
        procs = max(1, (os.cpu_count() or 8) // max(world, 1))
        self.mode = "classic"
        if a.config == "c2":
            seeds = range(rank * a.files, (rank + 1) * a.files)
            self.texts = make_texts("c2", seeds, a.file_bytes, procs)
            self.paths = [f"c2/r{rank}/f{s:07d}.cu" for s in seeds]
            self.desc = f"C2: {a.files} seeded MiniCU files x ~{a.file_bytes // 1000} KB per GPU, classic, nvcc 12"
        elif a.config == "c3":
            self.texts = [synth.gen_chain(64, a.c3_structs)]
            self.paths = ["c3/chains.cu"]
            self.desc = f"C3: one unit, 64-deep template chains over {a.c3_structs} structs, classic, nvcc 12"
        elif a.config == "c4":
            # one unit: with N > 1 ranks the SAME unit is walked by all of them
            # (strong scaling; levels exchanged through NCCL all-gathers)
            self.texts = [synth.gen_callgraph(a.c4_funcs, 10, 7)]
            self.paths = ["c4/callgraph.cu"]
            self.mode = "sound"
            self.desc = (f"C4: one unit, {a.c4_funcs} functions x 10 random calls, sound, nvcc 12"
                         + (f", walked by {world} ranks (NCCL all-gather per level)" if world > 1 else ""))
        else:  # c5: a pool of distinct stressor files cycled to c5_gb per GPU
            pool_n = a.c5_pool
            seeds = range(rank * pool_n, (rank + 1) * pool_n)
            pool_t = make_texts("c5", seeds, a.file_bytes, procs)
            per = sum(len(t) for t in pool_t) / pool_n
            n = int(a.c5_gb * 1e9 / per)
            self.texts = [pool_t[i % pool_n] for i in range(n)]
            self.paths = [f"c5/r{rank}/u{i:07d}.cu" for i in range(n)]
            self.pool = pool_n
            self.desc = (f"C5: {n} units (~{a.c5_gb:g} GB) per GPU cycling {pool_n} distinct seeded "
                         f"lexer-stressor files (~1% malformed), classic, nvcc 12; each unit analysed "
                         f"independently, every byte packed, copied and lexed")
        self.nbytes = sum(len(t) for t in self.texts)


# ---------------------------------------------------------------------------
# NVML clocks sampled during the timed region

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
# the reference (pure Python, installed unmodified into baseline/_ref) and the
# oracle port (tests' checker) on host cores

def _ref_import():
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    import exspace  # noqa: F401
    from exspace import spacecheck, preprocess  # noqa: F401
    return exspace


def _ref_unit(args):
    """One unit through the reference's own public API (spacecheck.py:687-739)."""
    text, mode = args
    ex = _ref_import()
    from exspace.spacecheck import Mode, analyze
    from exspace.syntax.preprocess import CompileProfile
    t0 = time.perf_counter()
    a = analyze(text, "u.cu", CompileProfile(), Mode(mode))
    dt = time.perf_counter() - t0
    edges = sum(len(v) for w in a.walks.values() for v in w.edges.values())
    _ = ex
    return len(text.encode()), edges, sum(1 for d in a.diagnostics if d.code in STRAY), dt


def reference_kind():
    try:
        _ref_import()
        return "reference"
    except Exception:
        return "port"


def _port_unit(args):
    text, mode = args
    from oracle import exs_oracle as O  # the checker / baseline only
    t0 = time.perf_counter()
    r = O.analyze_unit(text, mode)
    dt = time.perf_counter() - t0
    return (len(text.encode()), O.edge_count(r),
            sum(1 for d in r.diagnostics if d[0] in STRAY), dt)


def cpu_reference(texts, mode: str, cores: int):
    """Time the reference over ``texts`` on ``cores`` processes."""
    fn = _ref_unit if reference_kind() == "reference" else _port_unit
    t0 = time.perf_counter()
    if cores <= 1:
        res = [fn((t, mode)) for t in texts]
    else:
        with mp.Pool(cores) as pool:
            res = pool.map(fn, [(t, mode) for t in texts], chunksize=1)
    dt = time.perf_counter() - t0
    nbytes = sum(r[0] for r in res)
    edges = sum(r[1] for r in res)
    cpu_s = sum(r[3] for r in res)
    return {"gbs": nbytes / dt / 1e9, "edges_per_s": edges / dt, "seconds": dt, "bytes": nbytes,
            "files": len(texts), "gbs_per_core": nbytes / cpu_s / 1e9 if cpu_s else None}


def _oracle_check(args):
    text, mode = args
    from oracle import exs_oracle as O  # the checker only
    return O.check(text, mode)


def parity_sample(analyses, texts, idx, mode, procs):
    """Compare the e2e run's ordered diagnostics of units ``idx`` with the
    oracle (pinned to the reference's golden vectors)."""
    with mp.Pool(procs) as pool:
        want = pool.map(_oracle_check, [(texts[i], mode) for i in idx], chunksize=1)
    bad = 0
    n_d = n_s = 0
    for i, w in zip(idx, want):
        got = [(d.code, d.loc.line, d.loc.col, d.message) for d in analyses[i].diagnostics]
        n_d += len(got)
        n_s += sum(1 for g in got if g[0] in STRAY)
        if got != w:
            bad += 1
    return {"files": len(idx), "mismatches": bad, "diagnostics": n_d, "stray": n_s,
            "checker": "oracle/exs_oracle.py (pinned to the reference's golden vectors)"}


def run_reference_arm(a, rank, world):
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    kind = reference_kind()
    n = (a.ref_files or max(cores * 8, 32)) if a.config in ("c2", "c5") else 1
    vals = []
    if a.config in ("c2", "c5"):
        # the files the GPU arm times (rank 0's seeds), a window per step
        pool = a.files if a.config == "c2" else a.c5_pool
        for i in range(a.warmup + a.steps):
            seeds = [(i * n + j) % pool for j in range(n)]
            texts = make_texts(a.config, seeds, a.file_bytes, cores)
            r = cpu_reference(texts, "classic", cores)
            if i >= a.warmup:
                vals.append(r)
        sample = (f"{n} of the timed {a.config.upper()} files (~{n * a.file_bytes / 1e6:.1f} MB) per step, "
                  f"{'the reference package (baseline/_ref) exspace.analyze' if kind == 'reference' else 'oracle port'}"
                  f" over {cores} processes")
        workload = f"{a.config.upper()} sample of the GPU arm's files, classic, nvcc 12"
    else:
        small = {"c3": synth.gen_chain(64, 512), "c4": synth.gen_callgraph(100_000, 10, 7)}[a.config]
        mode = "sound" if a.config == "c4" else "classic"
        for i in range(max(1, min(a.steps, 2))):
            vals.append(cpu_reference([small], mode, 1))
        sample = ({"c3": "one unit of 64-deep chains over 512 structs",
                   "c4": "one unit of 100k functions x 10 calls (C4 scaled down 100x)"}[a.config] +
                  f", {'reference package' if kind == 'reference' else 'oracle port'} on 1 core")
        workload = f"{a.config.upper()} scaled-down sample, 1 core"
        cores = 1
    gbs = statistics.mean(v["gbs"] for v in vals)
    eps = statistics.mean(v["edges_per_s"] for v in vals)
    ms = statistics.mean(v["seconds"] for v in vals) * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s",
        "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (seeded generators, paper_2309_03912_b200/synth.py)",
        "config": {"workload": workload, "files_per_step": n, "file_bytes": a.file_bytes},
        "edges_per_s": eps,
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": cores, "kind": kind, "sample": sample,
                         "gbs_per_core": statistics.mean(v["gbs_per_core"] or 0 for v in vals)},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm

def run_gpu_arm(a, rank, world, local):
    import torch
    from paper_2309_03912_b200 import _native
    from paper_2309_03912_b200 import exspace as X

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    W = Workload(a, rank, world)
    mode = W.mode
    prof = X.CompileProfile()
    cfgb = X.cfg_byte(prof, X.Mode(mode), X.TraitConfig())
    eng = X.Engine(local, batch_mib=a.batch_mib)
    h = eng.handle
    h.set_option(9, a.pipelines)
    sharded_unit = a.config == "c4" and world > 1
    if sharded_unit:
        from paper_2309_03912_b200.shard import make_allgather
        h.set_collective(rank, world, make_allgather(device=local))
    nbytes = W.nbytes
    resident = a.config != "c5"  # C5 (8 GB per GPU) is measured end to end only
    if resident:
        blob = b"".join(t.encode() for t in W.texts)
        offs = np.zeros(len(W.texts) + 1, dtype=np.uint64)
        offs[1:] = np.cumsum([len(t) for t in W.texts])
        dev = torch.frombuffer(bytearray(blob), dtype=torch.uint8).to(f"cuda:{local}")
        del blob
        cfg = np.full(len(W.texts), cfgb, dtype=np.uint8)
        torch.cuda.synchronize()

    def run_resident():
        h.run_device(dev.data_ptr(), nbytes, offs, cfg)
        return h.stats()

    units = list(zip(W.paths, W.texts))

    def run_e2e():
        t0 = time.perf_counter()
        res = X.analyze_corpus(units, prof, X.Mode(mode), device=local, engine=eng)
        return time.perf_counter() - t0, res

    steps, kern = [], {}
    clk_sum = None
    if resident:
        for _ in range(a.warmup):
            run_resident()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
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
        clk_sum = clk.summary()
        torch.cuda.synchronize()
    # e2e through the public API with host str units.  The warm-up keeps each
    # run's results alive until the next run returns, as the timed loop does,
    # so the library's two result buffer sets are allocated before timing
    res = None
    for _ in range(2 if a.config == "c5" else max(2, min(a.warmup, 3))):
        _, res = run_e2e()
    if dist:
        dist.barrier()
    e2e_t = []
    e2e_stats = []
    with ClockSampler(local) as clk2:
        for _ in range(a.steps if a.config != "c5" else max(1, min(a.steps, 2))):
            t, res = run_e2e()
            e2e_t.append(t)
            e2e_stats.append(eng.last_stats)
    if clk_sum is None:
        clk_sum = clk2.summary()
    d2h_b = int(eng.last_result_bytes)
    e2e_ms = statistics.mean(e2e_t) * 1e3
    mean_ms = statistics.mean(s["ms_total"] for s in steps) if steps else e2e_ms
    if dist:
        tt = torch.tensor([mean_ms, e2e_ms], device=f"cuda:{local}")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        mean_ms, e2e_ms = tt.tolist()
    st = steps[-1] if steps else e2e_stats[-1]
    # one unit across the ranks (C4, N > 1) is strong scaling: the job is the unit
    total_bytes = nbytes if sharded_unit else nbytes * world
    total_edges = st["callsites"] if sharded_unit else st["callsites"] * world
    e2e = total_bytes / (e2e_ms / 1e3) / 1e9
    value = total_bytes / (mean_ms / 1e3) / 1e9 if resident else e2e
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
        traffic_db = json.loads(tf.read_text()).get(a.config, {})
    lex_ms = statistics.mean(s["ms_lex"] for s in steps) if steps else None
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": mean_ms, "higher_is_better": True,
        "scaling": "strong" if sharded_unit else "weak",
        "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (seeded generators, paper_2309_03912_b200/synth.py)",
        "config": {"workload": W.desc, "config": a.config, "units_per_gpu": len(W.texts),
                   "bytes_per_gpu": nbytes,
                   "parallelism": (f"walk split over {world} ranks, NCCL all-gather per level" if sharded_unit
                                   else f"dp{world} (unit shards, no data-path collective)"),
                   "l2": "inputs larger than L2; no flush", "batch_mib": a.batch_mib, "pipelines": a.pipelines,
                   "value_path": ("exs_run_device (corpus resident in HBM)" if resident
                                  else "= e2e (streamed; the corpus exceeds one device batch)")},
        "edges_per_s": total_edges / (mean_ms / 1e3),
        "stats": {k: st[k] for k in ("tokens", "items", "functions", "instances", "callsites", "levels",
                                     "diagnostics", "retries")},
        "stage_ms": ({k: statistics.mean(s[k] for s in steps) for k in ("ms_lex", "ms_parse", "ms_sema", "ms_walk")}
                     if steps else None),
        "gpu_launches": int(sum(s["gpu_launches"] for s in steps)) if steps else int(sum(
            s["gpu_launches"] for s in e2e_stats)),
        "roofline": ({"bound": "hbm", "achieved": per_kernel[dom].get("achieved_gbs"),
                      "peak": HBM_PEAK, "unit": "GB/s", "frac": per_kernel[dom].get("frac"),
                      "traffic": traffic_db.get(dom, {}).get("dram_bytes_per_launch"),
                      "algorithmic_bytes": (algo[dom] / max(1.0, per_kernel[dom]["launches_per_step"])
                                            if dom in algo else None),
                      "kernel": dom, "launches_per_step": per_kernel[dom]["launches_per_step"],
                      "share_of_step": per_kernel[dom]["share"], "peak_source": HBM_PEAK_SRC,
                      "traffic_source": traffic_db.get(dom, {}).get("source")}
                     if dom else None),
        "roofline_lex_stage": ({"bound": "hbm", "achieved": (nbytes + 32 * st["tokens"]) / (lex_ms / 1e3) / 1e9,
                                "peak": HBM_PEAK, "unit": "GB/s",
                                "frac": (nbytes + 32 * st["tokens"]) / (lex_ms / 1e3) / 1e9 / HBM_PEAK,
                                "kernel": "lex stage K1-K3 (all launches)"} if lex_ms else None),
        "kernels": per_kernel,
        "e2e": {"value": e2e, "unit": "GB/s", "h2d_bytes_per_step": int(nbytes), "d2h_bytes_per_step": d2h_b,
                "path": "exspace.analyze_corpus(units: list[(path, str)]) -> list[Analysis] (lazy Diagnostics)",
                "ms_per_step": e2e_ms, "batches": int(e2e_stats[-1]["batches"]),
                "device_ms_per_step": statistics.mean(s["ms_total"] for s in e2e_stats)},
        "clocks": clk_sum,
    }
    if rank == 0 and not a.no_parity:
        procs = os.cpu_count() or 8
        if a.config in ("c2", "c5"):
            nunits = len(W.texts)
            idx = sorted({(k * 7919) % nunits for k in range(a.parity_files)})
        else:
            idx = [0] if a.config == "c3" else []
        if idx:
            line["parity"] = parity_sample(res, W.texts, idx, mode, procs)
        if a.config == "c5":
            # units that share a pool text must report the same diagnostics
            rows = lambda k: [(d.code, d.loc.line, d.loc.col, d.message) for d in res[k].diagnostics]  # noqa: E731
            same = all(rows(k) == rows(k % W.pool) for k in range(W.pool, len(W.texts), max(1, len(W.texts) // 97)))
            line["parity"]["repeats_consistent"] = same
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cores = os.cpu_count() or 1
        if a.config in ("c2", "c5"):
            sample = W.texts[: max(cores * 8, 64)]
            r = cpu_reference(sample, mode, cores)
            r1 = cpu_reference(W.texts[:2], mode, 1)
            line["cpu_baseline"] = {
                "value": r["gbs"], "unit": "GB/s", "cores": cores, "kind": reference_kind(),
                "sample": f"the first {r['files']} timed files ({r['bytes'] / 1e6:.1f} MB), "
                          f"reference package exspace.analyze (baseline/_ref) on {cores} processes, "
                          f"{r['seconds']:.1f} s",
                "one_core_gbs": r1["gbs"]}
        elif a.config == "c4":
            small = synth.gen_callgraph(100_000, 10, 7)
            r = cpu_reference([small], mode, 1)
            line["cpu_baseline"] = {
                "value": r["gbs"], "unit": "GB/s", "cores": 1, "kind": reference_kind(),
                "sample": f"one unit of 100k functions x 10 calls ({r['bytes'] / 1e6:.1f} MB), reference on 1 core, "
                          f"{r['seconds']:.1f} s; linear extrapolation to 10M functions: "
                          f"{r['seconds'] * a.c4_funcs / 100_000:.0f} s",
                "edges_per_s": r["edges_per_s"]}
        else:
            small = synth.gen_chain(64, 512)
            r = cpu_reference([small], mode, 1)
            line["cpu_baseline"] = {
                "value": r["gbs"], "unit": "GB/s", "cores": 1, "kind": reference_kind(),
                "sample": f"one unit of 64-deep chains over 512 structs, reference on 1 core, {r['seconds']:.1f} s",
                "edges_per_s": r["edges_per_s"]}
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
    ap.add_argument("--config", default="c2", choices=["c2", "c3", "c4", "c5"])
    ap.add_argument("--files", type=int, default=10_000)
    ap.add_argument("--file-bytes", type=int, default=100_000)
    ap.add_argument("--batch-mib", type=int, default=256)
    ap.add_argument("--pipelines", type=int, default=2, help="concurrent batch pipelines on the GPU (1-4)")
    ap.add_argument("--c3-structs", type=int, default=10_300)
    ap.add_argument("--c4-funcs", type=int, default=10_000_000)
    ap.add_argument("--c5-gb", type=float, default=8.0)
    ap.add_argument("--c5-pool", type=int, default=2000)
    ap.add_argument("--parity-files", type=int, default=64)
    ap.add_argument("--ref-files", type=int, default=0, help="reference arm: files per step (0: 8 per core)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    a = ap.parse_args()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={29500 + os.getpid() % 1000}",
               str(Path(__file__).resolve())] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    rank, world, local = dist_env()
    if a.impl == "reference":
        run_reference_arm(a, rank, world)
    else:
        run_gpu_arm(a, rank, world, local)


if __name__ == "__main__":
    main()
