"""CPU-only tests: C-ABI library exports, host-side logic (legality mirror,
message rendering, configuration packing, synthetic generators) and the
multi-process file sharding over gloo (world_size 2).  No GPU needed."""
import ctypes
import os
import re
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "exspace_b200.h"
LIB = ROOT / "paper_2309_03912_b200" / "libexspace_b200.so"


def _ensure_lib():
    if not LIB.exists():
        import __graft_entry__ as g
        g.build()
    return LIB


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_ensure_lib()))
    decls = re.findall(r"\b(exs_\w+)\s*\(", HEADER.read_text())
    assert len(set(decls)) >= 14
    for name in set(decls):
        assert hasattr(lib, name), name


def test_no_gpu_fails_loudly_without_fallback():
    """Without a visible GPU the engine raises instead of computing on the CPU."""
    code = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_2309_03912_b200 import _native\n"
            "try:\n    _native.Handle(0)\nexcept _native.NativeError as e:\n    print('ERR', e)\n"
            "else:\n    print('OK')\n") % str(ROOT)
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         timeout=300)
    _ensure_lib()
    assert out.stdout.startswith("ERR"), out.stdout + out.stderr


def test_legality_mirror_matches_reference_tables():
    from paper_2309_03912_b200.exspace import DEVICE, HOST, ExecSpace, Mode, legality
    G, HD = ExecSpace.Global, ExecSpace.HostDevice
    # the reference's 32-entry matrix (test_spacecheck.py:22-73), restated
    expect = {}
    for caller in (HOST, DEVICE):
        for callee in (HOST, DEVICE, G, HD):
            for kind in ("direct", "launch"):
                for relaxed in (False, True):
                    if kind == "launch":
                        code = "E1003" if caller is DEVICE else (None if callee is G else "E1004")
                    elif callee is G:
                        code = "E1004"
                    elif relaxed or callee in (HD, caller):
                        code = None
                    else:
                        code = "E1001" if caller is HOST else "E1002"
                    expect[(caller, callee, kind, relaxed)] = code
    for (caller, callee, kind, relaxed), code in expect.items():
        v = legality(caller, callee, kind, relaxed_constexpr=relaxed, callee_is_constexpr=relaxed)
        assert v.code == code
    hd_cases = [(Mode.CLASSIC, HOST, True, "W1101"), (Mode.CLASSIC, DEVICE, True, "W1102"),
                (Mode.FIDELITY, HOST, True, "W1101"), (Mode.FIDELITY, DEVICE, True, None),
                (Mode.SOUND, HOST, True, "E1101"), (Mode.SOUND, DEVICE, True, "E1102"),
                (Mode.SOUND, HOST, False, "W1101"), (Mode.SOUND, DEVICE, False, "W1102"),
                (Mode.PROPOSAL1, HOST, True, "W1101"), (Mode.PROPOSAL1, DEVICE, True, "W1102"),
                (Mode.PROPOSAL2, HOST, True, "E1501"), (Mode.PROPOSAL2, DEVICE, False, "W1502")]
    for mode, callee, reach, code in hd_cases:
        caller = DEVICE if callee is HOST else HOST
        v = legality(caller, callee, caller_from_hd=True, mode=mode, mismatched_side_reachable=reach)
        assert v.code == code
    with pytest.raises(ValueError):
        legality(G, HOST)


def test_message_renderer_spans_and_splices():
    from paper_2309_03912_b200.messages import Renderer, M_P_EXPECTED, M_LEX_CHAR, M_S_UNDEF_NAME
    import numpy as np
    text = b"vo\\\nid f( {}\n\x0c x"
    ren = Renderer(text, [0, len(text)], b"")
    # an identifier split by a backslash-newline renders spliced
    span = (0 << 32) | 6
    assert ren.span_text(span) == "void"
    rec = np.zeros(1, dtype=[("msg", "<u2"), ("code", "<u2"), ("a0", "<u8"), ("a1", "<u8"),
                             ("a2", "<u8"), ("a3", "<u4")])[0]
    rec["msg"], rec["code"], rec["a0"], rec["a1"] = M_P_EXPECTED, 1, 13, 0xFFFFFFFFFFFFFFFF
    assert ren.message(rec) == "expected ')', found 'end of input'"
    rec["msg"], rec["a0"] = M_LEX_CHAR, (text.index(b"\x0c") << 32) | 1
    assert ren.message(rec) == "unexpected character '\\x0c'"
    rec["msg"], rec["code"], rec["a0"], rec["a3"] = M_S_UNDEF_NAME, 3, (7 << 32) | 1, 0
    assert ren.message(rec) == 'undefined name "f"'


def test_config_byte_packing():
    from paper_2309_03912_b200.exspace import CompileProfile, Mode, TraitConfig, cfg_byte
    assert cfg_byte(CompileProfile(), Mode.CLASSIC, TraitConfig()) == 0
    assert cfg_byte(CompileProfile(relaxed_constexpr=True), Mode.SOUND, TraitConfig()) == 2 | 16
    assert cfg_byte(CompileProfile("plain", erase_specifiers=True), Mode.PROPOSAL2,
                    TraitConfig(True)) == 4 | 8 | 32 | 64
    with pytest.raises(ValueError):
        CompileProfile("plain", relaxed_constexpr=True)


def test_synthetic_generators_are_deterministic_and_valid():
    from oracle import exs_oracle as O
    from paper_2309_03912_b200 import synth
    assert synth.gen_c2_file(3, 5000) == synth.gen_c2_file(3, 5000)
    assert synth.gen_chain(4, 8) == synth.gen_chain(4, 8)
    t = synth.gen_c2_file(11, 4000)
    assert t.isascii() and t.count("int main()") == 1
    # the oracle accepts them: no parse/preprocessor errors
    for text in (t, synth.gen_chain(5, 6), synth.gen_callgraph(40, 3, 1), synth.gen_c5_file(2, 4000, 0.0)):
        assert not [d for d in O.check(text) if d[0] in ("E0001", "E0002")]


def test_shard_ranges_are_contiguous_and_balanced():
    from paper_2309_03912_b200.shard import shard_ranges
    sizes = [100, 1, 1, 1, 100, 50, 50, 0, 200]
    for world in (1, 2, 3, 4, 8):
        r = shard_ranges(sizes, world)
        assert len(r) == world and r[0][0] == 0 and r[-1][1] == len(sizes)
        assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
    r = shard_ranges([10] * 100, 4)
    assert [hi - lo for lo, hi in r] == [25, 25, 25, 25]
    assert shard_ranges([], 3) == [(0, 0), (0, 0), (0, 0)]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


WORKER = r"""
import os, sys, json
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import torch.distributed as dist
from oracle import exs_oracle as O
from paper_2309_03912_b200 import synth
from paper_2309_03912_b200.shard import analyze_sharded
from exs_testlib import oracle_results
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:{port}", rank=rank, world_size=world)
units = [(f"f{{i:03d}}.cu", synth.gen_c5_file(i, 1500 + 400 * (i % 5), 0.3)) for i in range(13)]
# the per-rank analysis: the oracle's results in the library's columnar layout
# stand in for the GPU engine on CPU; the gather is the code under test
res = analyze_sharded(units, rank, world, lambda shard: oracle_results(shard, "sound"))
if rank == 0:
    print(json.dumps([[(d.code, d.loc.file, d.loc.line, d.loc.col, d.message) for d in a.diagnostics]
                      for a in res]))
dist.destroy_process_group()
"""


def test_sharded_analysis_gathers_in_path_order_over_gloo():
    port = _free_port()
    code = WORKER.format(root=str(ROOT), tests=str(ROOT / "tests"), port=port)
    procs = []
    for rank in range(2):
        env = dict(os.environ, RANK=str(rank), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1",
                   CUDA_VISIBLE_DEVICES="")
        procs.append(subprocess.Popen([sys.executable, "-c", code], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=600) for p in procs]
    assert all(p.returncode == 0 for p in procs), outs
    import json
    got = json.loads(outs[0][0].strip().splitlines()[-1])
    from oracle import exs_oracle as O
    from paper_2309_03912_b200 import synth
    units = [(f"f{i:03d}.cu", synth.gen_c5_file(i, 1500 + 400 * (i % 5), 0.3)) for i in range(13)]
    want = [[[d[0], p, d[1], d[2], d[3]] for d in O.check(t, "sound")] for p, t in units]
    assert got == want


def test_bench_gpus_n_relaunches_one_rank_per_gpu():
    """`bench.py --gpus 2` without torchrun re-launches itself under
    torch.distributed.run (one process per GPU); the reference arm runs on
    rank 0 only and prints one line with n_gpus 2."""
    import json
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--impl", "reference",
                          "--steps", "1", "--warmup", "0", "--ref-files", "2", "--file-bytes", "3000"],
                         capture_output=True, text=True, env=env, timeout=600, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["cpu_baseline"]["kind"] in ("reference", "port")


SHARD_WORKER = r"""
import os, sys, json
sys.path.insert(0, @ROOT@); sys.path.insert(0, @TESTS@)
import torch.distributed as dist
from paper_2309_03912_b200 import exspace as X
from paper_2309_03912_b200.shard import analyze_unit_sharded
from shard_units import UNITS
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:@PORT@", rank=rank, world_size=world)
eng = X.Engine(0, @LIB@)
out = []
for name, text, mode in UNITS:
    a = analyze_unit_sharded(text, name, rank, world, mode=X.Mode(mode), engine=eng, want_walks=True)
    out.append(ROW(a))
if rank == 0:
    print(json.dumps(out))
dist.destroy_process_group()
"""

ROW_SRC = r"""
def ROW(a):
    rows = [[d.code, d.loc.line, d.loc.col, d.message, d.suppressed] for d in a.all_diagnostics]
    walks = {k.value: [w.n_instances, w.n_edges, w.n_demands, sorted(w.instances),
                       sorted([k2, v] for k2, v in w.edges.items()),
                       sorted([k2, d, l[0], l[1]] for k2, (d, l) in w.demands.items())]
             for k, w in a.walks.items()}
    return [rows, walks]
"""


def _emu_lib():
    lib = ROOT / "build" / "libexspace_emu.so"
    if not lib.exists():
        if subprocess.run(["make", "-C", str(ROOT / "tests" / "emu")], capture_output=True).returncode:
            pytest.skip("the EMU build needs nvcc")
    return lib


@pytest.mark.parametrize("world", [2, 3])
def test_one_unit_walk_sharded_over_gloo_equals_one_rank(world):
    """One unit walked by `world` ranks (exs_set_collective; shard.analyze_unit_sharded):
    each rank walks its share of every level's work items and the ranks exchange new
    instances, edge slots, launch seeds and diagnostics through a gloo all-gather.  The
    kernels' logic runs as host code (the EMU build of the same sources; tests/emu), so the
    exchange protocol is checked here on CPU: diagnostics, walk counts and walk keys equal the
    single-rank run on deep chains (65 levels), call graphs, stressors, sema-diagnostic units."""
    import json
    lib = _emu_lib()
    port = _free_port()
    code = (ROW_SRC + SHARD_WORKER).replace("@ROOT@", repr(str(ROOT))).replace("@TESTS@", repr(str(ROOT / "tests")))
    code = code.replace("@PORT@", str(port)).replace("@LIB@", repr(str(lib)))
    procs = []
    for rank in range(world):
        env = dict(os.environ, RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                   CUDA_VISIBLE_DEVICES="")
        procs.append(subprocess.Popen([sys.executable, "-c", code], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=900) for p in procs]
    assert all(p.returncode == 0 for p in procs), [o[1][-2000:] for o in outs]
    got = json.loads(outs[0][0].strip().splitlines()[-1])
    sys.path.insert(0, str(ROOT / "tests"))
    from shard_units import UNITS
    from paper_2309_03912_b200 import exspace as X
    ns = {}
    exec(ROW_SRC, ns)
    eng = X.Engine(0, str(lib))
    want = [ns["ROW"](eng.run_batch([(t, n, X.CompileProfile(), X.Mode(m), X.TraitConfig())], want_walks=True)[0])
            for n, t, m in UNITS]
    assert json.loads(json.dumps(want)) == got
