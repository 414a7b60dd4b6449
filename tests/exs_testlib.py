"""Shared helpers for the test suite (golden fixtures, canonical keys)."""
import gzip
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"
GOLDEN_GROUPS = ["corpus", "genunit", "snippets", "synthetic", "mutations"]

from oracle import exs_oracle as O  # noqa: E402


def load_golden(name):
    with gzip.open(GOLDEN / f"{name}.json.gz", "rt", encoding="utf-8") as fh:
        return json.load(fh)


def canon_val(v):
    if isinstance(v, O.Ty):
        return v.name + ("<" + ",".join(v.targs) + ">" if v.targs else "")
    return "HDC::" + v.v


def canon_key(key):
    """Canonical text of an oracle walk key (same form as make_golden.canon_key)."""
    if key[0] == "decl":
        owner, name, params, req, spaces = key[1]
        return f"decl|{owner}|{name}|{';'.join(params)}|{req}|{spaces}"
    owner, name, params, req, spaces = key[1]
    binds = ",".join(f"{k}={canon_val(v)}" for k, v in key[2])
    ot = canon_val(key[3]) if key[3] is not None else ""
    s = f"inst|{owner}|{name}|{';'.join(params)}|{req}|{spaces}|{binds}|{ot}"
    if len(key) > 4:
        s += "|" + key[4]
    return s
