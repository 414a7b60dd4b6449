"""``Analysis.walks[side].instances / .demands / .edges`` rendered from the GPU.

The reference keeps, per walk (one compile pass, one native side), the instance
map, the demand map and the legal-edge lists keyed by tuples
(spacecheck.py:183-221, 239-346, 585):

  ("decl", (owner, name, params, req, spaces))                     demand of a decl
  ("inst", (owner, name, params, req, spaces), bindings, owner_type)   demand of an instance
  ("inst", ..., owner_type, side)                                   instance key

with ``params`` / ``req`` the canonical text of nodes._p_type / _p_expr
(nodes.py:336-383) and ``spaces`` the specifier signature (sema.py:133-149,
proposal2 only).  This module renders those keys in one canonical string form
-- the ``canon_key`` of tests/golden/make_golden.py:

  decl|owner|name|p1;p2|req|spaces
  inst|owner|name|p1;p2|req|spaces|T=S<Dev>,h=HDC::Dev|Owner<Hst>[|side]

from the arrays the library exports for the last batch (include/exspace_b200.h:
decls, structs, instances, edge slots, AST nodes, tokens).  Rendering is lazy:
nothing is fetched or built unless a walk's keys are read.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

NONE = 0xFFFFFFFF
# csrc/exs_common.cuh NodeKind
(N_INT, N_STR, N_BOOL, N_HDCV, N_ARCH, N_NAME, N_TMP, N_TRAIT, N_MCONST, N_CALL, N_MCALL, N_SCALL,
 N_NOT, N_BIN, N_TYPE, N_TPARAM, N_PARAM) = range(1, 18)
N_FN, N_FNX, N_STRUCT = 25, 26, 27
CALL_STD = 1
FF_H, FF_D, FF_G, FF_HPRED, FF_DPRED = 1, 2, 4, 256, 512
FR_DUP = 1
V_TYPE, V_HDC = 1, 2
BUILTIN = {1: "void", 2: "int", 3: "bool", 4: "HDC"}
HDC = {1: "Hst", 2: "Dev", 3: "HstDev"}
OPS = {1: "||", 2: "&&", 3: "==", 4: "!="}
SIDES = ("host", "device")


@dataclass
class InstanceInfo:
    """One instance of a walk (spacecheck.py:183-210)."""
    key: str          # canonical instance key (with side)
    demand_key: str   # canonical demand key (without side)
    decl: int         # creating declaration (index into the batch's decls)
    side: str
    display: str
    first_loc: tuple  # (line, col) of the first creation
    spaces: object = None  # effective spaces: GLOBAL or frozenset of ExecSpace (Instance.spaces)


GLOBAL = "global"  # sema.py GLOBAL: the spaces of a __global__ instance


@dataclass
class StructInfo:
    """One struct declaration of a pass's AST (nodes.py StructDecl): the name, the
    struct-level specifier bits (1 host, 2 device, 4 global) and the member
    functions as (name, specifier bits) in declaration order."""
    name: str
    spec: int
    members: list
    line: int

    def member_functions(self) -> list:
        return [m for m, _ in self.members]


class BatchWalks:
    """The walk arrays of one batch, fetched on first use."""

    def __init__(self, handle, renderer, status, modes):
        self.h = handle
        self.ren = renderer
        self.status = status      # exspace pass status per (file, pass)
        self.modes = modes        # Mode per file
        self._loaded = False

    def _load(self):
        if self._loaded:
            return
        h = self.h
        self.decls = h.decls()
        self.structs = h.structs()
        self.inst = h.instances()
        self.edge_slots = h.edges()
        self.nodes = h.nodes()
        n_tok = int(h.stats()["tokens"])
        self.toks = h.token_range(0, n_tok)
        # display names come from the device (exs_describe): fetch them now,
        # before a later run replaces the batch on the device
        nd, ni = len(self.decls), len(self.inst)
        if nd + ni:
            ids = list(range(nd)) + list(range(ni))
            kinds = [1] * nd + [2] * ni
            descs = self.ren.describe(ids, kinds)
            for j, (ident, kind) in enumerate(zip(ids, kinds)):
                self.ren._desc_cache[(ident, kind)] = descs[j]
        self._sig: dict = {}
        self._ikey: dict = {}
        self._loaded = True

    # -- text of the AST --------------------------------------------------------
    def _text(self, t: int) -> str:
        k = self.toks[t]
        return self.ren.span_text((int(k["pos"]) << 32) | (int(k["end"]) - int(k["pos"])))

    def _list(self, first: int):
        out, i = [], first
        while i != NONE:
            out.append(i)
            i = int(self.nodes[i]["next"])
        return out

    def p_type(self, t: int) -> str:  # nodes.py:336-340
        nd = self.nodes[t]
        name = self._text(int(nd["tok"]))
        targs = self._list(int(nd["c0"])) if int(nd["kind"]) == N_TYPE else []
        if targs:
            inner = ", ".join(self.p_type(a) if int(self.nodes[a]["kind"]) == N_TYPE else self.p_expr(a)
                              for a in targs)
            return f"{name}< {inner} >"
        return name

    def _p_targs(self, first: int) -> str:  # nodes.py:343-347
        targs = self._list(first)
        if not targs:
            return ""
        inner = ", ".join(self.p_type(a) if int(self.nodes[a]["kind"]) == N_TYPE else self.p_expr(a)
                          for a in targs)
        return f"< {inner} >"

    def _p_args(self, first: int) -> str:
        return ", ".join(self.p_expr(a) for a in self._list(first))

    def p_expr(self, e: int) -> str:  # nodes.py:354-382
        nd = self.nodes[e]
        k, tok = int(nd["kind"]), int(nd["tok"])
        if k == N_INT:
            return str(int(self.toks[tok]["hv"]))
        if k == N_STR:
            return f'"{self._text(tok)}"'
        if k == N_BOOL:
            return "true" if int(nd["sub"]) else "false"
        if k == N_HDCV:
            return f"HDC::{HDC[int(nd['sub'])]}"
        if k == N_ARCH:
            return "cuda_arch"
        if k == N_NAME:
            return self._text(tok)
        if k == N_TMP:
            return f"{self.p_type(int(nd['c0']))}{{}}"
        if k == N_TRAIT:
            return f"hdc< {self.p_type(int(nd['c0']))} >"
        if k == N_MCONST:
            return f"{self.p_type(int(nd['c0']))}::{self._text(tok)}"
        if k == N_CALL:
            if int(nd["sub"]) == CALL_STD:
                return f"std::{self._text(int(nd['c0']))}({self._p_args(int(nd['c2']))})"
            return f"{self._text(tok)}{self._p_targs(int(nd['c1']))}({self._p_args(int(nd['c2']))})"
        if k == N_MCALL:
            return (f"{self.p_expr(int(nd['c0']))}.{self._text(tok)}{self._p_targs(int(nd['c1']))}"
                    f"({self._p_args(int(nd['c2']))})")
        if k == N_SCALL:
            return (f"{self.p_type(int(nd['c0']))}::{self._text(tok)}{self._p_targs(int(nd['c1']))}"
                    f"({self._p_args(int(nd['c2']))})")
        if k == N_NOT:
            return f"!{self.p_expr(int(nd['c0']))}"
        if k == N_BIN:
            return f"({self.p_expr(int(nd['c0']))} {OPS[int(nd['sub'])]} {self.p_expr(int(nd['c1']))})"
        raise TypeError(f"node kind {k} is not an expression")

    # -- keys ---------------------------------------------------------------------
    def sig(self, d: int, p2: bool) -> str:
        """signature_key (sema.py:144-149) as owner|name|params|req|spaces."""
        key = (d, p2)
        if key not in self._sig:
            dr = self.decls[d]
            fn = self.nodes[int(dr["node"])]
            fx = self.nodes[int(dr["node"]) + 1]
            owner = ""
            if int(dr["rec"]) != NONE:
                owner = self._text(int(self.nodes[int(self.structs[int(dr["rec"])]["node"])]["tok"]))
            name = self._text(int(fn["tok"]))
            params = ";".join(self.p_type(int(self.nodes[p]["c0"])) for p in self._list(int(fn["c1"])))
            req = self.p_expr(int(fx["c0"])) if int(fx["c0"]) != NONE else ""
            spaces = ""
            if p2:  # sema.py:133-141
                fl = int(fn["n"])
                if fl & FF_H:
                    spaces += "H" + (f"({self.p_expr(int(fx['c1']))})" if fl & FF_HPRED else "")
                if fl & FF_D:
                    spaces += "D" + (f"({self.p_expr(int(fx['c2']))})" if fl & FF_DPRED else "")
                if fl & FF_G:
                    spaces += "G"
            self._sig[key] = f"{owner}|{name}|{params}|{req}|{spaces}"
        return self._sig[key]

    def canon_val(self, p: str, r) -> str:
        k = int(r[f"{p}_k"])
        if k == V_HDC:
            return f"HDC::{HDC[int(r[f'{p}_x'])]}"
        rec = int(r[f"{p}_rec"])
        name = (self._text(int(self.nodes[int(self.structs[rec]["node"])]["tok"])) if rec != NONE
                else BUILTIN[int(r[f"{p}_bt"])])
        targ = int(r[f"{p}_targ"])
        return f"{name}<{HDC[targ]}>" if targ else name

    def inst_keys(self, i: int, p2: bool):
        """(instance key, demand key) of instance i."""
        if i not in self._ikey:
            r = self.inst[i]
            d = int(r["decl"])
            fn = self.nodes[int(self.decls[d]["node"])]
            binds = []
            for tp in self._list(int(fn["c0"])):
                v = "tb" if int(self.nodes[tp]["sub"]) == 0 else "hb"
                if int(r[f"{v}_k"]):
                    binds.append((self._text(int(self.nodes[tp]["tok"])), self.canon_val(v, r)))
            binds.sort(key=lambda kv: kv[0])
            ot = self.canon_val("ot", r) if int(r["ot_k"]) == V_TYPE else ""
            dk = f"inst|{self.sig(d, p2)}|{','.join(f'{a}={b}' for a, b in binds)}|{ot}"
            self._ikey[i] = (f"{dk}|{SIDES[int(r['side'])]}", dk)
        return self._ikey[i]

    def walk(self, f: int, p: int):
        """(instances, demands, edges) of walk (file f, pass p), reference shapes:
        instances {key: InstanceInfo}; demands {key: (display, (line, col))};
        edges {caller key: [callee keys in post-order]}."""
        self._load()
        from .exspace import DEVICE, HOST, Mode
        p2 = self.modes[f] is Mode.PROPOSAL2
        w = 2 * f + p
        view = int(self.status[w]["view"])
        demands: dict = {}
        for d in range(len(self.decls)):  # _all_decls order (spacecheck.py:256-257)
            dr = self.decls[d]
            if int(dr["view"]) != view or int(dr["flags"]) & FR_DUP:
                continue
            k = f"decl|{self.sig(d, p2)}"
            if k not in demands:
                t = self.toks[int(self.nodes[int(dr["node"])]["tok"])]
                demands[k] = (self.ren.display(d, 1), (int(t["line"]), int(t["col"])))
        ids = [i for i in range(len(self.inst)) if int(self.inst[i]["walk"]) == w]
        ids.sort(key=lambda i: int(self.inst[i]["ckey"]))  # creation (FIFO) order
        instances, edges = {}, {}
        for i in ids:
            r = self.inst[i]
            key, dk = self.inst_keys(i, p2)
            t = self.toks[int(r["at"])]
            loc = (int(t["line"]), int(t["col"]))
            disp = self.ren.display(i, 2)
            sp = int(r["spaces"])
            spaces = GLOBAL if sp & 4 else frozenset(s for b, s in ((1, HOST), (2, DEVICE)) if sp & b)
            instances[key] = InstanceInfo(key, dk, int(r["decl"]), SIDES[int(r["side"])], disp, loc,
                                          spaces)
            fn = self.nodes[int(self.decls[int(r["decl"])]["node"])]
            if int(fn["c0"]) != NONE or int(r["ot_k"]) == V_TYPE:  # spacecheck.py:345-346
                demands.setdefault(dk, (disp, loc))
        for i in ids:
            r = self.inst[i]
            if not int(r["ecnt"]):
                continue
            b, n = int(r["ebase"]), int(self.decls[int(r["decl"])]["ncalls"])
            callees = [self.inst_keys(int(c), p2)[0] for c in self.edge_slots[b:b + n] if int(c) != NONE]
            if callees:
                edges[self.inst_keys(i, p2)[0]] = callees
        return instances, demands, edges

    def structs_of(self, f: int, p: int) -> list:
        """The struct declarations of (file f, pass p) in source order, each with
        its member functions (sema.py _all_decls records owned by the struct)."""
        self._load()
        view = int(self.status[2 * f + p]["view"])
        out, by_rec = [], {}
        for r in range(len(self.structs)):
            if int(self.structs[r]["view"]) == view:
                nd = self.nodes[int(self.structs[r]["node"])]
                t = self.toks[int(nd["tok"])]
                by_rec[r] = StructInfo(self._text(int(nd["tok"])), int(nd["n"]) & 7, [], int(t["line"]))
                out.append(by_rec[r])
        if by_rec:
            for d in np.nonzero(np.isin(self.decls["rec"], list(by_rec)))[0]:
                fn = self.nodes[int(self.decls[d]["node"])]
                by_rec[int(self.decls[d]["rec"])].members.append((self._text(int(fn["tok"])), int(fn["n"]) & 7))
        return out
