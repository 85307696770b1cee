"""Lowers a nest function (kernel-subset C) to sm_100a device code.

This is the backend's compile stage for the execution path: it takes a nest
text — the ORIGINAL source (nests/<nest>.c) or a form EMITTED by host stage
(a), this repo's re-implementation of the reference optimizer
(paper_2306_13002_b200/emitted/<nest>.<variant>.c, written by stage_a.py; the
``optimize_source`` contract of proj/src/pipeline.cpp:140-194) — and produces,
per registered region, a ``__device__`` per-point body.  The hand-written
kernel skeletons (csrc/kernels/*.cuh) decide the thread mapping and where each
array element comes from (global memory, a shared-memory tile, a register
queue, a warp shuffle); the body only names *which* element it needs.

Arithmetic is emitted with explicit IEEE round-to-nearest intrinsics so the
result never depends on nvcc's contraction choices:

* every ``+ - * /`` of the text is one rounding (``__dadd_rn`` …), in the
  text's evaluation order (C left-to-right, proj/src/printer.cpp precedence);
* in the saturated forms every extracted FMA temp ``_vN = a + b * c``
  (an ``Fma`` node, printed by proj/src/printer.cpp:114-125) becomes ONE
  ``__fma_rn(b, c, a)`` — the hardware FMA the paper's rules introduce
  (FMA1-3, proj/src/rules.cpp:129-135);
* C semantics of the reference interpreter otherwise (apply_bin/apply_un/
  apply_call/coerce, proj/src/interp.cpp:24-112): int∘int stays int with
  truncating ``/ %``, mixed operands promote to double, comparisons yield int,
  assignments coerce to the target type, sqrt is correctly rounded.

Loads: each array reference becomes ``m.template ld<ARR, o...>()`` when every
subscript is (loop variable + constant) or a constant — resolved through the
single-assignment ``_v`` int temps the emitter introduces (``_v4 = k + 1``) —
and ``m.template ldx<ARR>(idx...)`` otherwise (data-dependent donor/upwind
indices).  Stores likewise (``st`` / ``stx``).  In the ORIGINAL form the
skeleton issues one real global load per reference, in source order; in the
saturated forms loads are the CSE'd set the extraction kept.
"""
from __future__ import annotations

import os
import re
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

from . import kernel_subset as ks
from . import stage_a

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

LIBM1 = {"sqrt", "fabs", "sin", "cos", "exp", "log", "floor", "ceil"}
LIBM2 = {"pow", "fmin", "fmax"}


@dataclass
class Affine:
    var: Optional[str]   # loop variable, or None for a constant
    off: int


@dataclass
class Lowered:
    function: str
    params: List[ks.Param]
    loop_vars: List[str]
    bounds: List[Tuple[str, str]]             # per loop: (lo expr, hi expr), half-open, device C
    sig: Dict[str, List[int]]                 # array -> per position loop index / -1 absolute
    stored: set
    body: str                                 # device function body text
    n_fma: int = 0
    n_loads: int = 0
    n_dyn_loads: int = 0
    offrange: Dict[str, List[List[int]]] = field(default_factory=dict)
    ldrange: Dict[str, List[List[int]]] = field(default_factory=dict)
    dynrange: Dict[str, list] = field(default_factory=dict)
    dynsig: Dict[str, List[int]] = field(default_factory=dict)
    loaded: set = field(default_factory=set)
    # unconditional static stores: (array, per-position offset) written at
    # EVERY point of the iteration space on every path (both arms of an if)
    must_write: set = field(default_factory=set)
    # component slices: independent groups of stores (and the statements
    # they need), each emitted as its own device body; [] = not sliceable
    slices: List[str] = field(default_factory=list)
    slice_refs: List[list] = field(default_factory=list)   # per slice: sorted static load refs
    static_refs: set = field(default_factory=set)    # distinct (array, offsets) of static loads
    static_stores: set = field(default_factory=set)  # distinct (array, offsets) of static stores


class LowerError(Exception):
    pass


def ks_vars(e: Optional[ks.Expr]) -> set:
    """Scalar names an expression reads (array subscripts included)."""
    if e is None:
        return set()
    out = {e.op} if e.kind == "var" else set()
    for k in e.kids:
        out |= ks_vars(k)
    return out


def _affine_expr(var: Optional[str], off: int) -> ks.Expr:
    lit = ks.Expr("int", text=str(abs(off)))
    if var is None:
        return ks.Expr("int", text=str(off))
    v = ks.Expr("var", var)
    if off == 0:
        return v
    return ks.Expr("bin", "+" if off > 0 else "-", [v, lit])


class _Lowerer:
    def __init__(self, fn: ks.Function, region: ks.Region, fma: bool, f32: bool, ifconv: bool = True,
                 plain: bool = False):
        self.fn = fn
        self.region = region
        self.fma = fma
        self.f32 = f32
        self.types: Dict[str, str] = {}        # scalar name -> int|double
        self.arrays: Dict[str, ks.Param] = {}
        for p in fn.params:
            if p.dims:
                self.arrays[p.name] = p
            else:
                self.types[p.name] = p.ty
        self.loop_vars = [l.loop_var for l in region.marked_loops]
        if len(region.marked_loops) != len(region.loops):
            raise LowerError(f"{fn.name}: unmarked loops enclosing the region are not supported")
        for v in self.loop_vars:
            self.types[v] = "int"
        self.affine: Dict[str, Affine] = {v: Affine(v, 0) for v in self.loop_vars}
        self.assign_count: Dict[str, int] = {}
        self.sig: Dict[str, List[Optional[int]]] = {}
        self.offrange: Dict[str, List[List[int]]] = {}
        self.ldrange: Dict[str, List[List[int]]] = {}     # static LOADS only
        self.dynrange: Dict[str, List[Optional[List[int]]]] = {}  # value-set hints of ldx
        self.dynsig: Dict[str, List[int]] = {}
        self.int_assigns: Dict[str, List[ks.Expr]] = {}
        self.loaded = set()
        self.stored = set()
        self.n_fma = self.n_loads = self.n_dyn = 0
        self.capture: Optional[Dict[tuple, str]] = None   # if-conversion: store target -> value var
        self.capture_pair: Optional[Dict[tuple, str]] = None   # first arm's values (second arm stores)
        self.n_ifc = 0
        self.seq_vars: set = set()      # scalars assigned inside sequential inner loops
        self.ifconv = ifconv
        self.plain = plain      # nvcc-default arithmetic: C operators, contraction left to the compiler
        self.body_stmt: Optional[ks.Stmt] = None
        self.static_refs: set = set()
        self.static_stores: set = set()
        self.cur_refs: Optional[set] = None
        self.dead: set = set()          # ids of assignments under never-true guards
        self.slice_refs: List[list] = []

    # -- types
    def real(self) -> str:
        return "float" if self.f32 else "double"

    def expr_type(self, e: ks.Expr) -> str:
        if e.kind == "int":
            return "int"
        if e.kind == "float":
            return "double"
        if e.kind == "var":
            if e.op not in self.types:
                raise LowerError(f"undeclared scalar {e.op}")
            return self.types[e.op]
        if e.kind == "ref":
            return "int" if self.arrays[e.op].ty == "int" else "double"
        if e.kind == "call":
            return "double"
        if e.kind == "un":
            return "int" if e.op == "!" else self.expr_type(e.kids[0])
        if e.op in ("<", "<=", ">", ">=", "==", "!=", "&&", "||"):
            return "int"
        a, b = self.expr_type(e.kids[0]), self.expr_type(e.kids[1])
        return "int" if a == b == "int" else "double"

    # -- affine resolution of subscripts
    def count_assigns(self, s: ks.Stmt, in_loop: bool = False):
        if s.kind == "assign" and s.lhs.kind == "var":
            self.assign_count[s.lhs.op] = self.assign_count.get(s.lhs.op, 0) + 1
            if in_loop:
                self.seq_vars.add(s.lhs.op)   # assigned in a sequential loop: no static value set
            elif id(s) not in self.dead:      # never executed: no candidate value
                self.int_assigns.setdefault(s.lhs.op, []).append(s.rhs)
        for c in ks.children(s):
            self.count_assigns(c, in_loop or s.kind == "for")
        if s.kind == "assign" and s.lhs.kind == "var" and s.lhs.op in self.seq_vars:
            self.int_assigns.pop(s.lhs.op, None)

    @staticmethod
    def assigned_in(s: ks.Stmt) -> set:
        out = set()
        if s.kind == "assign" and s.lhs.kind == "var":
            out.add(s.lhs.op)
        for c in ks.children(s):
            out |= _Lowerer.assigned_in(c)
        return out

    # -- guards the loop bounds decide ---------------------------------------
    #
    # advec's `if (upwind > nx - 1) upwind = nx - 1;` follows `upwind = j + 1`
    # inside `for (j = 2; j < nx - 2; j++)`: j + 1 <= nx - 2 < nx - 1, so the
    # clamp never runs and upwind's candidate values are {j - 2, j + 1} — all
    # affine in j, so its loads can be served from the staged box unchecked.
    # Symbolic linear forms over loop variables and scalar parameters
    # ({name: coeff}, const); a guard is dead when its comparison is false at
    # every point of the iteration space.

    def lin(self, e: ks.Expr, env) -> Optional[Tuple[Dict[str, int], int]]:
        if e.kind == "int":
            return {}, int(e.text)
        if e.kind == "var":
            if e.op in env:
                return env[e.op]
            if e.op in self.loop_vars or (self.types.get(e.op) == "int" and e.op in self.fn_param_names):
                return {e.op: 1}, 0
            return None
        if e.kind == "bin" and e.op in ("+", "-"):
            a, b = self.lin(e.kids[0], env), self.lin(e.kids[1], env)
            if a is None or b is None:
                return None
            sg = 1 if e.op == "+" else -1
            co = dict(a[0])
            for k, v in b[0].items():
                co[k] = co.get(k, 0) + sg * v
            return {k: v for k, v in co.items() if v}, a[1] + sg * b[1]
        return None

    def always_false(self, cond: ks.Expr, env) -> bool:
        """cond (a < b, a <= b, a > b, a >= b) false at every iteration-space point."""
        if cond.kind != "bin" or cond.op not in ("<", "<=", ">", ">="):
            return False
        a, b = self.lin(cond.kids[0], env), self.lin(cond.kids[1], env)
        if a is None or b is None:
            return False
        # d = a - b; the guard holds when d > 0 (>), d >= 0 (>=), d < 0 (<), d <= 0 (<=)
        co = dict(a[0])
        for k, v in b[0].items():
            co[k] = co.get(k, 0) - v
        const = a[1] - b[1]
        co = {k: v for k, v in co.items() if v}
        want_pos = cond.op in (">", ">=")
        strict = cond.op in (">", "<")
        # extreme of d over the loop ranges: loop var v in [lo_v, hi_v - 1]
        ext, ext_c = {}, const
        for v, c in co.items():
            if v not in self.loop_ranges:
                ext[v] = ext.get(v, 0) + c       # parameters stay symbolic
                continue
            (lo, lo_c), (hi, hi_c) = self.loop_ranges[v]
            take_hi = (c > 0) == want_pos        # maximise d for >, minimise for <
            form, fc = (hi, hi_c - 1) if take_hi else (lo, lo_c)
            for k, w in form.items():
                ext[k] = ext.get(k, 0) + c * w
            ext_c += c * fc
        if any(w for w in ext.values()):
            return False                        # still depends on a parameter
        if want_pos:
            return ext_c <= 0 if strict else ext_c < 0
        return ext_c >= 0 if strict else ext_c > 0

    def find_dead(self, s: ks.Stmt, env, out: set):
        """Walk the body in order, tracking int scalars with linear values;
        collect the assignments under guards that can never hold."""
        k = s.kind
        if k == "block":
            for c in s.stmts:
                self.find_dead(c, env, out)
        elif k == "assign" and s.lhs.kind == "var":
            v = self.lin(s.rhs, env)
            if v is not None:
                env[s.lhs.op] = v
            else:
                env.pop(s.lhs.op, None)
        elif k == "for":
            # a sequential inner loop: every scalar it assigns has no single
            # linear value afterwards (and none inside: the body repeats)
            for name in self.assigned_in(s):
                env.pop(name, None)
        elif k == "if":
            if self.always_false(s.cond, env):
                self.mark_dead(s.then_s, out)
                if s.else_s is not None:
                    self.find_dead(s.else_s, env, out)
                return
            e1, e2 = dict(env), dict(env)
            self.find_dead(s.then_s, e1, out)
            if s.else_s is not None:
                self.find_dead(s.else_s, e2, out)
            for name in set(e1) | set(e2) | set(env):   # keep only values both arms agree on
                if e1.get(name) == e2.get(name) and name in e1:
                    env[name] = e1[name]
                else:
                    env.pop(name, None)

    def mark_dead(self, s: ks.Stmt, out: set):
        if s.kind == "assign":
            out.add(id(s))
        for c in ks.children(s):
            self.mark_dead(c, out)

    def as_affine(self, e: ks.Expr) -> Optional[Affine]:
        if e.kind == "int":
            return Affine(None, int(e.text))
        if e.kind == "var":
            return self.affine.get(e.op)
        if e.kind == "bin" and e.op in ("+", "-"):
            a, b = self.as_affine(e.kids[0]), self.as_affine(e.kids[1])
            if a is None or b is None:
                return None
            if e.op == "+" and (a.var is None or b.var is None):
                return Affine(a.var or b.var, a.off + b.off)
            if e.op == "-" and b.var is None:
                return Affine(a.var, a.off - b.off)
        return None

    def ref_offsets(self, e: ks.Expr) -> Optional[List[int]]:
        arr = e.op
        offs, sig = [], []
        for idx in e.kids:
            a = self.as_affine(idx)
            if a is None:
                return None
            sig.append(self.loop_vars.index(a.var) if a.var is not None else -1)
            offs.append(a.off)
        known = self.sig.get(arr)
        if known is None:
            self.sig[arr] = sig
        elif known != sig:
            return None        # inconsistent position mapping: go dynamic
        rng = self.offrange.setdefault(arr, [[o, o] for o in offs])
        for p, o in enumerate(offs):
            rng[p][0] = min(rng[p][0], o)
            rng[p][1] = max(rng[p][1], o)
        return offs

    # -- expressions
    def lit(self, e: ks.Expr) -> str:
        t = e.text.rstrip("fF")
        if self.f32:
            return t + "f" if ("." in t or "e" in t or "E" in t) else t
        return t

    def conv(self, code: str, have: str, want: str) -> str:
        if have == want:
            return code
        if want == "double":
            return f"(({self.real()})({code}))"
        return f"((int)({code}))"

    def ex(self, e: ks.Expr) -> Tuple[str, str]:
        k = e.kind
        if k == "int":
            return e.text, "int"
        if k == "float":
            return self.lit(e), "double"
        if k == "var":
            return e.op, self.types[e.op]
        if k == "ref":
            return self.load(e), ("int" if self.arrays[e.op].ty == "int" else "double")
        if k == "call":
            return self.call(e), "double"
        if k == "un":
            c, t = self.ex(e.kids[0])
            if e.op == "!":
                return f"(!({c}))", "int"
            return f"(-({c}))", t
        op = e.op
        if op in ("&&", "||"):
            a, _ = self.ex(e.kids[0])
            b, _ = self.ex(e.kids[1])
            return f"(({a}) {op} ({b}))", "int"
        a, ta = self.ex(e.kids[0])
        b, tb = self.ex(e.kids[1])
        if ta == tb == "int":
            if op in ("/", "%"):
                # C truncation semantics (interp: int /0 and %0 are EvalErrors)
                return f"(({a}) {op} ({b}))", "int"
            return f"(({a}) {op} ({b}))", "int"
        a, b = self.conv(a, ta, "double"), self.conv(b, tb, "double")
        if op in ("<", "<=", ">", ">=", "==", "!="):
            return f"(({a}) {op} ({b}))", "int"
        if op == "%":
            raise LowerError("'%' requires integer operands")
        if self.plain:
            return f"(({a}) {op} ({b}))", "double"
        sfx = "f" if self.f32 else "d"
        name = {"+": "add", "-": "sub", "*": "mul", "/": "div"}[op]
        return f"__{sfx}{name}_rn({a}, {b})", "double"

    def call(self, e: ks.Expr) -> str:
        args = [self.conv(*self.ex(a), "double") for a in e.kids]
        n = e.op
        f = "f" if self.f32 else ""
        if n == "sqrt":
            if self.plain:
                return f"sqrt{f}({args[0]})"
            return f"__{'f' if self.f32 else 'd'}sqrt_rn({args[0]})"
        if n in LIBM1 and len(args) == 1:
            return f"{n}{f}({args[0]})"
        if n in LIBM2 and len(args) == 2:
            return f"{n}{f}({args[0]}, {args[1]})"
        raise LowerError(f"unknown function {n}/{len(args)}")

    def value_set(self, e: ks.Expr, seen=None) -> List[Optional[Affine]]:
        """Possible affine values of an int subscript expression (None = not
        affine in the loop variables).  Used only as a HINT for which box of a
        dynamically indexed array a tile should stage; the kernels re-check
        every dynamic index at run time."""
        seen = set() if seen is None else seen
        a = self.as_affine(e)
        if a is not None:
            return [a]
        if e.kind == "var" and e.op in self.int_assigns and e.op not in seen:
            seen = seen | {e.op}
            out: List[Optional[Affine]] = []
            for rhs in self.int_assigns[e.op]:
                out.extend(self.value_set(rhs, seen))
            return out
        if e.kind == "bin" and e.op in ("+", "-"):
            ls, rs = self.value_set(e.kids[0], seen), self.value_set(e.kids[1], seen)
            out = []
            for x in ls:
                for y in rs:
                    if x is None or y is None:
                        out.append(None)
                    elif e.op == "+" and (x.var is None or y.var is None):
                        out.append(Affine(x.var or y.var, x.off + y.off))
                    elif e.op == "-" and y.var is None:
                        out.append(Affine(x.var, x.off - y.off))
                    else:
                        out.append(None)
            return out
        return [None]

    def record_dynamic(self, e: ks.Expr):
        arr = e.op
        sig, rng = [], []
        for idx in e.kids:
            vals = [v for v in self.value_set(idx) if v is not None]
            vars_ = {v.var for v in vals}
            if not vals or len(vars_) != 1:
                sig.append(-2)        # unknown: no staging for this position
                rng.append(None)
                continue
            var = vars_.pop()
            sig.append(self.loop_vars.index(var) if var is not None else -1)
            rng.append([min(v.off for v in vals), max(v.off for v in vals)])
        old = self.dynsig.get(arr)
        if old is not None and old != sig:
            sig = [a if a == b else -2 for a, b in zip(old, sig)]
        self.dynsig[arr] = sig
        cur = self.dynrange.setdefault(arr, [None] * len(rng))
        for p, r in enumerate(rng):
            if sig[p] == -2 or r is None:
                cur[p] = None
            elif cur[p] is None:
                cur[p] = list(r)
            else:
                cur[p] = [min(cur[p][0], r[0]), max(cur[p][1], r[1])]

    def load(self, e: ks.Expr) -> str:
        self.n_loads += 1
        self.loaded.add(e.op)
        offs = self.ref_offsets(e)
        arr = f"ARR_{e.op}"
        if offs is not None:
            r = self.ldrange.setdefault(e.op, [[o, o] for o in offs])
            for p, o in enumerate(offs):
                r[p][0] = min(r[p][0], o)
                r[p][1] = max(r[p][1], o)
            self.static_refs.add((e.op, tuple(offs)))
            if self.cur_refs is not None:
                self.cur_refs.add((e.op, tuple(offs)))
            return f"m.template ld<{arr}, {', '.join(str(o) for o in offs)}>()"
        self.record_dynamic(e)
        self.n_dyn += 1
        idx = ", ".join(self.conv(*self.ex(i), "int") for i in e.kids)
        # every candidate value of every subscript affine in ONE loop variable
        # (or constant): the tiled skeletons size their staged box to hold all
        # of them, so the element needs no range check (ldx_in)
        safe = True
        for i in e.kids:
            vals = self.value_set(i)
            if any(v is None for v in vals) or len({v.var for v in vals}) != 1:
                safe = False
        return f"m.template {'ldx_in' if safe else 'ldx'}<{arr}>({idx})"

    # -- statements
    def is_fma_temp(self, s: ks.Stmt) -> Optional[Tuple[ks.Expr, ks.Expr, ks.Expr]]:
        if not (self.fma and s.lhs.kind == "var" and s.lhs.op.startswith("_v")):
            return None
        r = s.rhs
        if r.kind == "bin" and r.op == "+" and r.kids[1].kind == "bin" and r.kids[1].op == "*":
            a, (b, c) = r.kids[0], r.kids[1].kids
            atoms = ("var", "int", "float")

            def atom(x):
                return x.kind in atoms or (x.kind == "un" and x.op == "-" and x.kids[0].kind in atoms)
            if atom(a) and atom(b) and atom(c) and self.types.get(s.lhs.op) == "double":
                return a, b, c
        return None

    def st(self, s: ks.Stmt, ind: int, out: List[str]):
        pad = "    " * ind
        k = s.kind
        if k == "decl":
            for name, dims, init in s.names:
                if dims:
                    raise LowerError("local arrays are not supported on the device path")
                self.types[name] = s.ty
                ty = "int" if s.ty == "int" else self.real()
                if init is not None:
                    c = self.conv(*self.ex(init), s.ty)
                    out.append(f"{pad}{ty} {name} = {c};")
                else:
                    out.append(f"{pad}{ty} {name};")
            return
        if k == "assign":
            fm = self.is_fma_temp(s)
            if s.lhs.kind == "var":
                name = s.lhs.op
                if name not in self.types:
                    raise LowerError(f"assignment to undeclared {name}")
                tgt = self.types[name]
                if fm:
                    a, b, c = (self.conv(*self.ex(x), "double") for x in fm)
                    self.n_fma += 1
                    fn = "__fmaf_rn" if self.f32 else "__fma_rn"
                    out.append(f"{pad}{name} = {fn}({b}, {c}, {a});")
                    return
                code, t = self.ex(s.rhs)
                out.append(f"{pad}{name} = {self.conv(code, t, tgt)};")
                # int temps defined once by an affine expression resolve subscripts statically
                if tgt == "int" and self.assign_count.get(name, 0) == 1 and name not in self.loop_vars:
                    a = self.as_affine(s.rhs)
                    if a is not None:
                        self.affine[name] = a
                return
            if s.lhs.kind == "ref":
                arr = s.lhs.op
                self.stored.add(arr)
                want = "int" if self.arrays[arr].ty == "int" else "double"
                code, t = self.ex(s.rhs)
                val = self.conv(code, t, want)
                offs = self.ref_offsets(s.lhs)
                if self.capture is not None:    # if-converted branch: the store becomes a value
                    key = self.target_key(s.lhs)
                    out.append(f"{pad}{self.capture[key]} = {val};")
                    if self.capture_pair is not None:
                        # second arm: store the selected element right away, so
                        # its value is not held until the end of the arm
                        out.append(f"{pad}m.template st<ARR_{arr}, {', '.join(map(str, offs))}>"
                                   f"(_ifc ? {self.capture_pair[key]} : {self.capture[key]});")
                    return
                if offs is not None:
                    self.static_stores.add((arr, tuple(offs)))
                    out.append(f"{pad}m.template st<ARR_{arr}, {', '.join(map(str, offs))}>({val});")
                else:
                    idx = ", ".join(self.conv(*self.ex(i), "int") for i in s.lhs.kids)
                    out.append(f"{pad}m.template stx<ARR_{arr}>({idx}, {val});")
                return
            raise LowerError("bad assignment target")
        if k == "if":
            targets = self.if_convertible(s)
            if targets is not None:
                self.if_convert(s, targets, ind, out)
                return
            c, _ = self.ex(s.cond)
            out.append(f"{pad}if ({c}) {{")
            self.st(s.then_s, ind + 1, out)
            if s.else_s is not None:
                out.append(f"{pad}}} else {{")
                self.st(s.else_s, ind + 1, out)
            out.append(f"{pad}}}")
            return
        if k == "block":
            out.append(f"{pad}{{")
            for c in s.stmts:
                self.st(c, ind + 1, out)
            out.append(f"{pad}}}")
            return
        if k == "empty":
            return
        if k == "call":
            out.append(f"{pad}(void){self.call(s.call)};")
            return
        if k == "for":
            # a sequential loop inside the per-point body (an unmarked inner
            # loop: matmul's k, a scan): the thread runs it as written; its
            # variable is never a static subscript, so loads indexed by it are
            # dynamic (ldx) and its stores conditional (not must-write)
            if s.init is not None:
                self.st(s.init, ind, out)
            c, _ = self.ex(s.cond) if s.cond is not None else ("1", "int")
            out.append(f"{pad}while ({c}) {{")
            self.st(s.body, ind + 1, out)
            if s.step is not None:
                self.st(s.step, ind + 1, out)
            out.append(f"{pad}}}")
            return
        raise LowerError(f"statement kind {k}")

    # -- if-conversion of store-symmetric branches
    #
    # In the bulk-load forms the reference emitter hoists every load above the
    # branch (proj/src/codegen.cpp:429-495), which can leave an `if` whose two
    # arms are load-free and store to the SAME set of elements — D3Q19's
    # obstacle bounce-back vs BGK collide arms both write the 19 pushed
    # distributions.  On a SIMT machine a warp holding both kinds of cell
    # would issue every store twice with complementary lane masks; instead
    # both arms are evaluated (pure arithmetic, no traps on the GPU) and each
    # element is stored ONCE with a select of the two values.  Bit-exact: the
    # stored value is the one the taken arm computes.

    def target_key(self, e: ks.Expr) -> Optional[tuple]:
        offs = []
        for idx in e.kids:
            a = self.as_affine(idx)
            if a is None:
                return None
            offs.append((a.var, a.off))
        return (e.op, tuple(offs))

    @staticmethod
    def _has_ref(e: Optional[ks.Expr]) -> bool:
        if e is None:
            return False
        return e.kind == "ref" or any(_Lowerer._has_ref(k) for k in e.kids)

    def _arm(self, s: ks.Stmt, targets: list, assigned: set, reads: set, local: set) -> bool:
        k = s.kind
        if k == "empty":
            return True
        if k == "block":
            return all(self._arm(c, targets, assigned, reads, local) for c in s.stmts)
        if k == "decl":
            for name, dims, init in s.names:
                if dims or self._has_ref(init):
                    return False
                local.add(name)
                if init is not None:
                    reads.update(ks_vars(init))
            return True
        if k == "assign":
            if self._has_ref(s.rhs):
                return False
            reads.update(ks_vars(s.rhs))
            if s.lhs.kind == "var":
                assigned.add(s.lhs.op)
                return True
            if s.lhs.kind == "ref" and not any(self._has_ref(i) for i in s.lhs.kids):
                key = self.target_key(s.lhs)
                if key is None:
                    return False
                targets.append(key)
                return True
        return False

    def if_convertible(self, s: ks.Stmt) -> Optional[list]:
        if not self.ifconv or s.else_s is None:
            return None
        ta, tb = [], []
        aa, ab, ra, rb, la, lb = set(), set(), set(), set(), set(), set()
        if not (self._arm(s.then_s, ta, aa, ra, la) and self._arm(s.else_s, tb, ab, rb, lb)):
            return None
        if not ta or sorted(ta, key=repr) != sorted(tb, key=repr) or len(set(ta)) != len(ta):
            return None
        # scalars an arm assigns that live outside it: neither arm may read the
        # other's, and nothing after the `if` may read them (they would see
        # both arms' writes)
        outer_a, outer_b = aa - la, ab - lb
        if (outer_a & rb) or (outer_b & ra):
            return None
        if (outer_a | outer_b) & self.reads_outside(s):
            return None
        return ta

    def reads_outside(self, target: ks.Stmt) -> set:
        out: set = set()

        def walk(st: ks.Stmt):
            if st is target:
                return
            for e in (st.rhs, st.cond, st.lhs if st.lhs is not None and st.lhs.kind == "ref" else None):
                if e is not None:
                    out.update(ks_vars(e))
            for _, _, init in st.names:
                if init is not None:
                    out.update(ks_vars(init))
            for c in ks.children(st):
                walk(c)
        walk(self.body_stmt)
        return out

    def if_convert(self, s: ks.Stmt, targets: list, ind: int, out: List[str]):
        pad = "    " * ind
        ty = {}
        for key in targets:
            ty[key] = "int" if self.arrays[key[0]].ty == "int" else self.real()
        names_a = {key: f"_ifc{self.n_ifc}_a{i}" for i, key in enumerate(targets)}
        names_b = {key: f"_ifc{self.n_ifc}_b{i}" for i, key in enumerate(targets)}
        self.n_ifc += 1
        c, _ = self.ex(s.cond)
        out.append(f"{pad}{{  // if-converted: both arms store the same {len(targets)} elements")
        out.append(f"{pad}    const bool _ifc = ({c});")
        for key in targets:
            out.append(f"{pad}    {ty[key]} {names_a[key]}, {names_b[key]};")
        for key in targets:
            if any(v is not None and v not in self.loop_vars for v, _ in key[1]):
                raise LowerError("if-conversion target not in loop coordinates")
        saved = (self.capture, self.capture_pair)
        self.capture, self.capture_pair = names_a, None
        self.st(s.then_s, ind + 1, out)
        # the second arm stores each element (one select) as soon as it is computed
        self.capture, self.capture_pair = names_b, names_a
        self.st(s.else_s, ind + 1, out)
        self.capture, self.capture_pair = saved
        out.append(f"{pad}}}")

    def must_write(self, s: ks.Stmt) -> set:
        """Store targets executed on every path through `s` (static offsets
        only; a loop var position gives its offset, an absolute position its
        constant).  Evaluated after emission, so int temps are resolved."""
        k = s.kind
        if k == "block":
            out = set()
            for c in s.stmts:
                out |= self.must_write(c)
            return out
        if k == "if":
            if s.else_s is None:
                return set()
            return self.must_write(s.then_s) & self.must_write(s.else_s)
        if k == "assign" and s.lhs.kind == "ref":
            key = self.target_key(s.lhs)
            if key is None:
                return set()
            sig = self.sig.get(key[0])
            offs = tuple(o for _, o in key[1])
            vars_ = [v for v, _ in key[1]]
            want = [self.loop_vars[i] if i is not None and i >= 0 else None for i in (sig or [])]
            if sig is None or vars_ != want:
                return set()
            return {(key[0], offs)}
        return set()

    # -- component slicing
    #
    # zsolve's 75 stores fall into 25 groups (one per 5x5 block entry m, n)
    # that share no loaded element: lhsZ[m][n][*] reads only fjacZ[m][n] and
    # njacZ[m][n].  Each group, with the statements its stores need (scalar
    # temps duplicated), is an independent per-point body, so the skeleton can
    # spread components over threads: 25x the parallelism, 1/25 of the live
    # state per thread.  Exact: every stored value is computed by the same
    # statements in the same order.

    def _flat(self, s: ks.Stmt, out: List[ks.Stmt]) -> bool:
        if s.kind == "block":
            return all(self._flat(c, out) for c in s.stmts)
        if s.kind in ("decl", "assign", "empty"):
            out.append(s)
            return True
        return False

    def _fields(self, e: Optional[ks.Expr], out: set):
        if e is None:
            return
        if e.kind == "ref":
            key = []
            for p, idx in enumerate(e.kids):
                a = self.as_affine(idx)
                if a is None:
                    key = None
                    break
                if a.var is None:
                    key.append((p, a.off))
            out.add((e.op, tuple(key) if key is not None else None))
        for k in e.kids:
            self._fields(k, out)

    def slice_groups(self) -> Optional[List[List[ks.Stmt]]]:
        stmts: List[ks.Stmt] = []
        if not self._flat(self.body_stmt, stmts):
            return None
        names = [n for s_ in stmts if s_.kind == "decl" for n, _, _ in s_.names]
        if len(names) != len(set(names)):
            return None
        assigns = [s_ for s_ in stmts if s_.kind == "assign"]
        defs: Dict[str, ks.Stmt] = {}
        for s_ in assigns:
            if s_.lhs.kind == "var":
                if s_.lhs.op in defs:
                    return None                    # multiply-assigned scalar: keep whole
                defs[s_.lhs.op] = s_
        stores = [s_ for s_ in assigns if s_.lhs.kind == "ref"]
        if len(stores) < 2 or (self.stored & self.loaded):
            return None
        order = {id(s_): i for i, s_ in enumerate(stmts)}
        memo: Dict[int, set] = {}

        def back(st: ks.Stmt) -> set:
            if id(st) in memo:
                return memo[id(st)]
            out = {id(st)}
            used = ks_vars(st.rhs) | (ks_vars(st.lhs) if st.lhs.kind == "ref" else set())
            for v in used:
                if v in defs:
                    out |= back(defs[v])
            memo[id(st)] = out
            return out

        by_id = {id(s_): s_ for s_ in stmts}
        parent = list(range(len(stores)))

        def find(a):
            while parent[a] != a:
                parent[a] = parent[parent[a]]
                a = parent[a]
            return a
        owner: Dict[tuple, int] = {}
        for i, st in enumerate(stores):
            f: set = set()
            for sid in back(st):
                self._fields(by_id[sid].rhs, f)
                if by_id[sid].lhs.kind == "ref":
                    for idx in by_id[sid].lhs.kids:
                        self._fields(idx, f)
            for key in f:
                if key in owner:
                    parent[find(i)] = find(owner[key])
                else:
                    owner[key] = i
        groups: Dict[int, set] = {}
        for i, st in enumerate(stores):
            groups.setdefault(find(i), set()).update(back(st))
        if len(groups) < 2:
            return None
        decls = [s_ for s_ in stmts if s_.kind == "decl"]
        out = []
        import copy
        for root in sorted(groups, key=lambda r: min(order[x] for x in groups[r])):
            ids = sorted(groups[root], key=lambda x: order[x])
            body = [by_id[x] for x in ids]
            used = set()
            for st in body:
                used |= ks_vars(st.rhs) | ks_vars(st.lhs)
            kept = []
            for d in decls:            # only the temps this slice touches
                names = [nm for nm in d.names if nm[0] in used]
                if names:
                    d2 = copy.copy(d)
                    d2.names = names
                    kept.append(d2)
            out.append(kept + body)
        return out

    def emit_slices(self) -> List[str]:
        groups = self.slice_groups()
        if not groups:
            return []
        saved = (self.n_fma, self.n_loads, self.n_dyn)
        bodies = []
        for g in groups:
            out: List[str] = ["    " + x for x in self.pre]   # function-level locals (temp1, ...)
            self.cur_refs = set()
            for st in g:
                self.st(st, 2, out)
            self.slice_refs.append(sorted(self.cur_refs))
            self.cur_refs = None
            bodies.append("\n".join(out))
        self.n_fma, self.n_loads, self.n_dyn = saved
        return bodies

    def bound_expr(self, e: ks.Expr) -> str:
        c, t = self.ex(e)
        if t != "int":
            raise LowerError("loop bounds must be int")
        return c.replace("m.template", "<bad>")

    def loop_bounds(self) -> List[Tuple[str, str]]:
        out = []
        for l in self.region.loops:
            if l.init.kind != "assign" or l.cond is None or l.cond.kind != "bin":
                raise LowerError("unsupported loop header")
            step = l.step
            if not (step.kind == "assign" and step.rhs.kind == "bin" and step.rhs.op == "+"
                    and step.rhs.kids[1].kind == "int" and step.rhs.kids[1].text == "1"):
                raise LowerError("only unit-step loops are supported")
            lo = self.bound_expr(l.init.rhs)
            op = l.cond.op
            hi = self.bound_expr(l.cond.kids[1])
            if l.cond.kids[0].kind != "var" or l.cond.kids[0].op != l.loop_var:
                raise LowerError("loop condition must test the loop variable")
            if op == "<=":
                hi = f"({hi}) + 1"
            elif op != "<":
                raise LowerError("loop condition must be < or <=")
            out.append((lo, hi))
        return out

    def run(self) -> Lowered:
        body_stmt = self.region.anchor.body
        self.body_stmt = body_stmt
        # loop ranges as linear forms of the parameters (for dead guards)
        self.fn_param_names = {p.name for p in self.fn.params if not p.dims}
        self.loop_ranges = {}
        for l in self.region.loops:
            lo = self.lin(l.init.rhs, {}) if l.init is not None and l.init.kind == "assign" else None
            hi = self.lin(l.cond.kids[1], {}) if l.cond is not None and l.cond.kind == "bin" else None
            if lo is not None and hi is not None and l.cond.op in ("<", "<="):
                if l.cond.op == "<=":
                    hi = (hi[0], hi[1] + 1)
                self.loop_ranges[l.loop_var] = (lo, hi)
        self.find_dead(body_stmt, {}, self.dead)
        self.count_assigns(body_stmt)
        # function-level locals other than loop vars
        pre: List[str] = []

        def fn_level(stmts):
            for s in stmts:
                if s.kind == "decl":
                    for name, dims, init in s.names:
                        if name in self.loop_vars:
                            continue
                        if dims:
                            raise LowerError("local arrays are not supported")
                        self.types[name] = s.ty
                        ty = "int" if s.ty == "int" else self.real()
                        pre.append(f"    {ty} {name};")
                elif s.kind == "for":
                    if s is not self.region.loops[0]:
                        raise LowerError("only one loop nest per function is supported")
                elif s.kind == "block":
                    fn_level(s.stmts)          # `#pragma acc parallel { ... }` around the nest
                elif s.kind != "empty":
                    raise LowerError("statements outside the loop nest are not supported")
        fn_level(self.fn.body.stmts)
        for name in getattr(self, "global_scalars", ()):
            if self.assign_count.get(name):
                raise LowerError(f"the region assigns the global scalar '{name}' (a reduction): not offloaded")
        bounds = self.loop_bounds()
        self.pre = pre
        out: List[str] = list(pre)
        self.st(body_stmt, 1, out)
        must = self.must_write(body_stmt)
        slices = self.emit_slices()
        sig = {a: self.sig.get(a) for a in self.arrays}
        return Lowered(self.fn.name, self.fn.params, self.loop_vars, bounds,
                       {a: (s if s is not None else [-1] * len(self.arrays[a].dims)) for a, s in sig.items()},
                       self.stored, "\n".join(out), self.n_fma, self.n_loads, self.n_dyn, self.offrange,
                       self.ldrange, self.dynrange, self.dynsig, self.loaded, must, slices, self.slice_refs,
                       self.static_refs, self.static_stores)


def global_params(mod: ks.Module) -> List[ks.Param]:
    """File-scope declarations a region reads, as implicit parameters after the
    function's own (the caller passes the globals' storage / values)."""
    out = []
    for s in mod.globals:
        if s.kind == "decl":
            for name, dims, init in s.names:
                out.append(ks.Param(s.ty, name, list(dims)))
    return out


def _walk_stmts(s: Optional[ks.Stmt]):
    if s is None:
        return
    yield s
    for c in ks.children(s):
        yield from _walk_stmts(c)


def _stmt_reads_writes(s: ks.Stmt) -> Tuple[set, set]:
    """Scalar names a statement subtree reads / assigns (loop headers included)."""
    reads, writes = set(), set()
    for t in _walk_stmts(s):
        if t.kind == "assign":
            if t.lhs.kind == "var":
                writes.add(t.lhs.op)           # compound forms are desugared: x = x + e reads x
            else:
                for k in t.lhs.kids:
                    reads |= ks_vars(k)
            reads |= ks_vars(t.rhs)
        elif t.kind == "decl":
            for name, dims, init in t.names:
                reads |= ks_vars(init)
                if init is not None:
                    writes.add(name)
        for e in (t.cond, t.call):
            reads |= ks_vars(e)
    return reads, writes


def simple_nest_function(fn: ks.Function, region: ks.Region) -> bool:
    """The function body is declarations plus the region's loops, all marked
    (the shape every benchmark nest has: the region IS the function)."""
    if len(region.marked_loops) != len(region.loops):
        return False

    def ok(stmts):
        for s in stmts:
            if s.kind in ("decl", "empty") or s is region.loops[0]:
                continue
            if s.kind == "block" and ok(s.stmts):
                continue
            return False
        return True
    return ok(fn.body.stmts if fn.body.kind == "block" else [fn.body])


def region_view(mod: ks.Module, fn: ks.Function, region: ks.Region) -> Tuple[ks.Function, ks.Region, List[ks.Param]]:
    """The region as a function of its own: the marked nest only, with the
    scalars it takes from the enclosing function as implicit parameters —
    the variables of unmarked loops ENCLOSING the nest (a time loop around it
    runs on the host and passes its index per launch) and function locals the
    nest reads but never assigns (live-ins).  Returns (function, region,
    implicit params).  Unmarked loops must enclose the marked ones
    (the reference's iteration space, proj/src/ast.cpp:333-398)."""
    marked = region.marked_loops
    n_un = len(region.loops) - len(marked)
    if region.loops[n_un:] != marked:
        raise LowerError(f"{fn.name}: an unmarked loop between marked loops of the region")
    top = marked[0]
    decl_ty: Dict[str, str] = {}
    for t in _walk_stmts(fn.body):
        if t.kind == "decl":
            for name, dims, init in t.names:
                if not dims:
                    decl_ty[name] = t.ty
    known = {p.name for p in fn.params} | {p.name for p in global_params(mod)}
    implicit: List[ks.Param] = []
    for l in region.loops[:n_un]:
        if l.loop_var in known:
            raise LowerError(f"{fn.name}: enclosing loop variable '{l.loop_var}' is a parameter")
        implicit.append(ks.Param("int", l.loop_var, []))
    reads, writes = _stmt_reads_writes(top)
    inner_vars = {l.loop_var for l in marked}
    taken = {p.name for p in implicit}
    for name in sorted(reads - writes - inner_vars - known - taken):
        if name in decl_ty:
            implicit.append(ks.Param(decl_ty[name], name, []))
    # the nest's own temporaries stay local declarations of the view
    drop = {p.name for p in implicit}
    decls = []
    for name, ty in decl_ty.items():
        if name not in drop and name not in inner_vars and name in (reads | writes):
            decls.append(ks.Stmt("decl", ty=ty, names=[(name, [], None)]))
    body = ks.Stmt("block", stmts=decls + [top])
    vfn = ks.Function(fn.name, list(fn.params) + implicit, body)
    vreg = ks.Region(vfn, region.index, list(marked), region.anchor)
    return vfn, vreg, implicit


def region_params(mod: ks.Module, fn: ks.Function, region: Optional[ks.Region] = None) -> List[ks.Param]:
    """The kernel's parameters: the function's own, the file's globals, and —
    for a region that is not the whole function — its implicit parameters
    (region_view)."""
    own = {p.name for p in fn.params}
    out = list(fn.params) + [p for p in global_params(mod) if p.name not in own]
    if region is not None and not simple_nest_function(fn, region):
        out += region_view(mod, fn, region)[2]
    return out


def lower_text(text: str, function: str, fma: bool, f32: bool = False, ifconv: bool = True,
               plain: bool = False, region_index: Optional[int] = None) -> Lowered:
    """Lowers the region of `function` (the one with `region_index`, the
    module-wide find_regions index, when the function has several)."""
    mod = ks.parse(text)
    for reg in ks.find_regions(mod):
        if reg.function.name == function and (region_index is None or reg.index == region_index):
            fn0 = reg.function
            if not simple_nest_function(fn0, reg):
                fn0, reg, _ = region_view(mod, fn0, reg)
            fn = ks.Function(fn0.name, region_params(mod, fn0), fn0.body)
            low = _Lowerer(fn, reg, fma, f32, ifconv, plain)
            low.global_scalars = {p.name for p in global_params(mod) if not p.dims}
            return low.run()
    raise LowerError(f"no region in function {function}")


# ---------------------------------------------------------------------------
# Header generation

FORMS = [("original", None, False), ("cse", "cse", False), ("cse_bulk", "cse+bulk", False),
         ("cse_sat", "cse+sat", True), ("accsat", "accsat", True)]


def _scalar_struct(params, f32):
    real = "float" if f32 else "double"
    lines = ["struct Scalars {"]
    for p in params:
        if not p.dims:
            lines.append(f"    {'int' if p.ty == 'int' else real} {p.name};")
    lines.append("};")
    return lines


def gen_function(nest: str, function: str, f32: bool = False, sources: Optional[Dict[str, str]] = None,
                 region_index: Optional[int] = None, ns_name: Optional[str] = None) -> Tuple[str, dict]:
    """Device bodies of every form of one nest function (of its region
    `region_index` when it has several; the struct is then named `ns_name`).
    `sources` maps each form's variant (None = the original) to its module
    text; default: the benchmark nest's text and host stage (a)'s emitted files."""
    ns = (ns_name or function) + ("_f32" if f32 else "")
    texts = {}
    for form, variant, fma in FORMS:
        if sources is not None:
            texts[form] = (sources[variant], fma)
            continue
        path = os.path.join(ROOT, "nests", f"{nest}.c") if variant is None else stage_a.ensure(nest, variant)
        texts[form] = (open(path).read(), fma)
    lows = {form: lower_text(t, function, fma, f32, region_index=region_index) for form, (t, fma) in texts.items()}
    base = lows["original"]
    arrays = [p for p in base.params if p.dims]
    # merge signatures across forms (all forms must agree on static position maps)
    sig = {}
    for a in arrays:
        cands = [l.sig[a.name] for l in lows.values() if any(x != -1 for x in l.sig[a.name])]
        sig[a.name] = cands[0] if cands else [-1] * len(a.dims)
        for c in cands:
            if c != sig[a.name]:
                raise LowerError(f"{function}: forms disagree on the position map of {a.name}")
    stored = set().union(*(l.stored for l in lows.values()))
    L = []
    L.append(f"struct {ns} {{")
    L.extend(_scalar_struct(base.params, f32))
    L.append("enum : int {")
    for i, a in enumerate(arrays):
        L.append(f"    ARR_{a.name} = {i},")
    L.append(f"    NARR = {len(arrays)}")
    L.append("};")
    L.append(f"static constexpr int NLOOP = {len(base.loop_vars)};")
    L.append(f"static constexpr int MAXDIM = 8;")
    L.append("// per array, per subscript position: index of the loop variable it is")
    L.append("// relative to (0 = outermost marked loop), or -1 = absolute constant")
    rows = ", ".join("{" + ", ".join(str(x) for x in (sig[a.name] + [-1] * (8 - len(a.dims)))) + "}"
                     for a in arrays)
    L.append(f"static __host__ __device__ constexpr int sig(int a, int p) {{ constexpr int t[NARR][8] = {{{rows}}}; return t[a][p]; }}")
    L.append("static __host__ __device__ constexpr int ndim(int a) { constexpr int t[NARR] = {"
             + ", ".join(str(len(a.dims)) for a in arrays) + "}; return t[a]; }")
    L.append("// arrays never stored by any form: safe for the read-only (ld.global.nc) path")
    L.append("static __host__ __device__ constexpr bool readonly(int a) { constexpr bool t[NARR] = {"
             + ", ".join("false" if a.name in stored else "true" for a in arrays) + "}; return t[a]; }")
    L.append("static __host__ __device__ constexpr bool is_int(int a) { constexpr bool t[NARR] = {"
             + ", ".join("true" if a.ty == "int" else "false" for a in arrays) + "}; return t[a]; }")
    L.append("static constexpr const char* array_names[NARR] = {" + ", ".join(f'"{a.name}"' for a in arrays) + "};")
    sc = [p for p in base.params if not p.dims]
    L.append(f"static constexpr int NSCALAR = {len(sc)};")
    L.append("static constexpr const char* scalar_names[NSCALAR] = {" + ", ".join(f'"{p.name}"' for p in sc) + "};")
    L.append("static constexpr bool scalar_is_int[NSCALAR] = {" + ", ".join("true" if p.ty == "int" else "false" for p in sc) + "};")
    L.append("static inline void set_scalar(Scalars& s, int idx, long long iv, double dv) {")
    L.append("    switch (idx) {")
    for i, p in enumerate(sc):
        L.append(f"        case {i}: s.{p.name} = {'(int)iv' if p.ty == 'int' else ('(float)dv' if f32 else 'dv')}; break;")
    L.append("    }")
    L.append("}")
    try:
        inner_lo = int(base.bounds[-1][0])
    except ValueError:
        inner_lo = -999
    L.append(f"static constexpr int inner_lo_const = {inner_lo};   // innermost loop's lower bound if constant, else -999")
    L.append("// iteration space: half-open [lo, hi) per marked loop, outermost first")
    L.append("static __host__ __device__ inline void bounds(const Scalars& s, long long lo[NLOOP], long long hi[NLOOP]) {")
    for p in sc:
        L.append(f"    const auto {p.name} = s.{p.name}; (void){p.name};")
    for d, (lo, hi) in enumerate(base.bounds):
        L.append(f"    lo[{d}] = {lo}; hi[{d}] = {hi};")
    L.append("}")
    meta = {}
    # measurement baseline (acs_variant 5, ACS_ORIGINAL_NVCC): the original text
    # as nvcc compiles it by default — C operators with FMA contraction left to
    # the compiler, loads free to be cached/CSE'd.  Not bit-exact by design.
    nv = lower_text(texts["original"][0], function, False, f32, plain=True, region_index=region_index)
    lvn = ", ".join(f"const int {v}" for v in nv.loop_vars)
    L.append("// form original_nvcc: the original text, nvcc-default arithmetic (contraction allowed)")
    L.append("template <class M>")
    L.append(f"static __device__ __forceinline__ void body_original_nvcc(M& m, const Scalars& s_, {lvn}) {{")
    for p in sc:
        ty = "int" if p.ty == "int" else ("float" if f32 else "double")
        L.append(f"    {ty} {p.name} = s_.{p.name}; (void){p.name};")
    L.append(nv.body)
    L.append("}")
    for form, low in lows.items():
        lv = ", ".join(f"const int {v}" for v in low.loop_vars)
        L.append(f"// form {form}: {low.n_loads} static loads ({low.n_dyn_loads} data-dependent), "
                 f"{low.n_fma} single-rounding FMA")
        L.append(f"template <class M>")
        L.append(f"static __device__ __forceinline__ void body_{form}(M& m, const Scalars& s_, {lv}) {{")
        for p in sc:
            ty = "int" if p.ty == "int" else ("float" if f32 else "double")
            L.append(f"    {ty} {p.name} = s_.{p.name}; (void){p.name};")
        L.append(low.body)
        L.append("}")
        meta[form] = {"loads": low.n_loads, "dyn_loads": low.n_dyn_loads, "fma": low.n_fma,
                      "slices": max(1, len(low.slices))}
        L.append(f"// form {form}: {max(1, len(low.slices))} independent component slice(s)")
        L.append(f"template <int SLICE, class M>")
        L.append(f"static __device__ __forceinline__ void body_{form}_slice(M& m, const Scalars& s_, {lv}) {{")
        if low.slices:
            for p in sc:
                ty = "int" if p.ty == "int" else ("float" if f32 else "double")
                L.append(f"    {ty} {p.name} = s_.{p.name}; (void){p.name};")
            for si, b in enumerate(low.slices):
                L.append(f"    {'if' if si == 0 else 'else if'} constexpr (SLICE == {si}) {{")
                L.append(b)
                L.append("    }")
        else:
            L.append(f"    body_{form}(m, s_, {', '.join(low.loop_vars)});")
        L.append("}")
    forms = [f for f, _, _ in FORMS]
    L.append("// per acs_variant (ORIGINAL, CSE, CSE_BULK, CSE_SAT, ACCSAT)")
    L.append("static constexpr int static_loads[5] = {" + ", ".join(str(meta[f]["loads"]) for f in forms) + "};")
    L.append("static constexpr int fma_count[5] = {" + ", ".join(str(meta[f]["fma"]) for f in forms) + "};")
    # static offset range per array/position over every form (host-side bounds check)
    rng = {}
    for low in lows.values():
        for a, r in low.offrange.items():
            cur = rng.setdefault(a, [list(x) for x in r])
            for p, (lo_, hi_) in enumerate(r):
                cur[p][0] = min(cur[p][0], lo_)
                cur[p][1] = max(cur[p][1], hi_)
    rows_lo, rows_hi = [], []
    for a in arrays:
        r = rng.get(a.name, [[0, 0]] * len(a.dims))
        rows_lo.append("{" + ", ".join(str(x[0]) for x in r + [[0, 0]] * (8 - len(r))) + "}")
        rows_hi.append("{" + ", ".join(str(x[1]) for x in r + [[0, 0]] * (8 - len(r))) + "}")
    L.append("// min / max static subscript offset per array and position (all forms)")
    L.append("static constexpr int off_lo[NARR][8] = {" + ", ".join(rows_lo) + "};")
    L.append("static constexpr int off_hi[NARR][8] = {" + ", ".join(rows_hi) + "};")
    # staging tables: per array/position, the box of LOADED elements relative to the
    # point (static loads + value-set hints of data-dependent loads)
    stage = {}
    for a in arrays:
        nd = len(a.dims)
        sg = list(sig[a.name])
        lo_ = [None] * nd
        hi_ = [None] * nd
        ok = True
        for low in lows.values():
            if a.name in low.ldrange:
                for p, (x, y) in enumerate(low.ldrange[a.name]):
                    lo_[p] = x if lo_[p] is None else min(lo_[p], x)
                    hi_[p] = y if hi_[p] is None else max(hi_[p], y)
            if a.name in low.dynsig:
                ds, dr = low.dynsig[a.name], low.dynrange[a.name]
                for p in range(nd):
                    if ds[p] == -2 or dr[p] is None:
                        ok = False
                        continue
                    if all(v == -1 for v in sig[a.name]) and not any(a.name in l.ldrange for l in lows.values()):
                        sg[p] = ds[p]
                    elif ds[p] != sg[p]:
                        ok = False
                        continue
                    lo_[p] = dr[p][0] if lo_[p] is None else min(lo_[p], dr[p][0])
                    hi_[p] = dr[p][1] if hi_[p] is None else max(hi_[p], dr[p][1])
        loaded = any(a.name in l.loaded for l in lows.values())
        # an array written by the nest is never staged: a staged copy could be
        # stale after the thread's own store (load-after-store, e.g. the
        # original advec re-reads mass_flux_x)
        stage[a.name] = (loaded and ok and a.name not in stored and all(v is not None for v in lo_), sg,
                         [v if v is not None else 0 for v in lo_], [v if v is not None else 0 for v in hi_])
    def row(vals):
        return "{" + ", ".join(str(x) for x in list(vals) + [0] * (8 - len(vals))) + "}"
    L.append("// staging (TMA) tables: loaded box per array/position relative to the point")
    L.append("static __host__ __device__ constexpr bool stageable(int a) { constexpr bool t[NARR] = {"
             + ", ".join("true" if stage[a.name][0] else "false" for a in arrays) + "}; return t[a]; }")
    L.append("static __host__ __device__ constexpr bool is_loaded(int a) { constexpr bool t[NARR] = {"
             + ", ".join("true" if any(a.name in l.loaded for l in lows.values()) else "false" for a in arrays)
             + "}; return t[a]; }")
    L.append("static __host__ __device__ constexpr int ld_sig(int a, int p) { constexpr int t[NARR][8] = {"
             + ", ".join("{" + ", ".join(str(x) for x in stage[a.name][1] + [-1] * (8 - len(a.dims))) + "}" for a in arrays)
             + "}; return t[a][p]; }")
    L.append("static __host__ __device__ constexpr int ld_lo(int a, int p) { constexpr int t[NARR][8] = {"
             + ", ".join(row(stage[a.name][2]) for a in arrays) + "}; return t[a][p]; }")
    L.append("static __host__ __device__ constexpr int ld_hi(int a, int p) { constexpr int t[NARR][8] = {"
             + ", ".join(row(stage[a.name][3]) for a in arrays) + "}; return t[a][p]; }")
    must = set.intersection(*(l.must_write for l in lows.values()))
    names = [a.name for a in arrays]
    must = sorted(must, key=lambda t: (names.index(t[0]), t[1]))
    L.append("// unconditional static stores of EVERY form (array, offsets): written at every point")
    L.append(f"static constexpr int n_must_write = {len(must)};")
    L.append("static constexpr int must_write_arr[" + str(max(1, len(must))) + "] = {"
             + (", ".join(f"ARR_{a}" for a, _ in must) if must else "-1") + "};")
    L.append("static constexpr int must_write_off[" + str(max(1, len(must))) + "][8] = {"
             + (", ".join(row(list(o)) for _, o in must) if must else row([])) + "};")
    # register-window rows (march skeleton, several adjacent x points per
    # thread): distinct (array, subscript offsets except the innermost-loop
    # position) of the static loads of every form, with the x-offset range
    nl = len(base.loop_vars)
    rowmap: Dict[tuple, List[int]] = {}
    used: Dict[tuple, set] = {}
    for fi, (form, low) in enumerate(lows.items()):
        for arr, offs in low.static_refs:
            sg = sig[arr]
            xp = sg.index(nl - 1) if (nl - 1) in sg else -1
            key = (names.index(arr), tuple(o if p != xp else 0 for p, o in enumerate(offs)))
            ox = offs[xp] if xp >= 0 else 0
            r = rowmap.setdefault(key, [ox, ox])
            r[0], r[1] = min(r[0], ox), max(r[1], ox)
            used.setdefault(key, set()).add(fi)
    rkeys = sorted(rowmap)
    L.append("// register-window rows: static-load rows (array, offsets with the innermost-loop position")
    L.append("// zeroed), their x-offset range, and which forms (bit per acs_variant) read them")
    L.append(f"static constexpr int NROW = {len(rkeys)};")
    def tab(name, vals):
        vals = list(vals) or [0]
        L.append(f"static __host__ __device__ constexpr int {name}(int r) {{ constexpr int t[{len(vals)}] = {{"
                 + ", ".join(str(v) for v in vals) + "}; return t[r]; }")
    tab("row_arr", [k[0] for k in rkeys])
    tab("row_xlo", [rowmap[k][0] for k in rkeys])
    tab("row_xhi", [rowmap[k][1] for k in rkeys])
    tab("row_forms", [sum(1 << f for f in used[k]) for k in rkeys])
    offs_rows = [row(list(k[1])) for k in rkeys] or [row([])]
    L.append(f"static __host__ __device__ constexpr int row_off(int r, int p) {{ constexpr int t[{len(offs_rows)}][8] = {{"
             + ", ".join(offs_rows) + "}; return t[r][p]; }")
    # store rows: distinct static store targets of every form (deferred
    # vector stores of a thread's adjacent points)
    srow: Dict[tuple, set] = {}
    for fi, (form, low) in enumerate(lows.items()):
        for arr, offs in low.static_stores:
            srow.setdefault((names.index(arr), offs), set()).add(fi)
    skeys = sorted(srow)
    L.append(f"static constexpr int NSROW = {len(skeys)};")
    tab("srow_arr", [k[0] for k in skeys])
    tab("srow_forms", [sum(1 << f for f in srow[k]) for k in skeys])
    soffs = [row(list(k[1])) for k in skeys] or [row([])]
    L.append(f"static __host__ __device__ constexpr int srow_off(int r, int p) {{ constexpr int t[{len(soffs)}][8] = {{"
             + ", ".join(soffs) + "}; return t[r][p]; }")
    # per (form, slice): its static load refs (register queue of the sliced skeleton)
    refl = []          # flattened (arr, offs)
    start = []         # per form*MAXS + slice: first index
    count = []
    maxs = max(meta[f]["slices"] for f in forms)
    for f in forms:
        low = lows[f]
        per = low.slice_refs if low.slices else [sorted(low.static_refs)]
        for si in range(maxs):
            refs = per[si] if si < len(per) else []
            start.append(len(refl))
            count.append(len(refs))
            refl.extend(refs)
    L.append(f"static constexpr int MAXSLICE = {maxs};")
    L.append("static __host__ __device__ constexpr int sl_first(int f, int s) { constexpr int t[] = {"
             + ", ".join(map(str, start)) + "}; return t[f * MAXSLICE + s]; }")
    L.append("static __host__ __device__ constexpr int sl_nref(int f, int s) { constexpr int t[] = {"
             + ", ".join(map(str, count)) + "}; return t[f * MAXSLICE + s]; }")
    L.append("static __host__ __device__ constexpr int sl_arr(int i) { constexpr int t[] = {"
             + (", ".join(str(names.index(a)) for a, _ in refl) or "0") + "}; return t[i]; }")
    L.append("static __host__ __device__ constexpr int sl_off(int i, int p) { constexpr int t[][8] = {"
             + (", ".join(row(list(o)) for _, o in refl) or row([])) + "}; return t[i][p]; }")
    L.append("static constexpr bool has_dynamic_index = " + ("true" if any(m_["dyn_loads"] for m_ in meta.values()) else "false") + ";")
    args = ", ".join(f"pt[{d}]" for d in range(len(base.loop_vars)))
    L.append("// component slices per acs_variant (1 = the whole body)")
    L.append("static constexpr int nslices[5] = {" + ", ".join(str(meta[f]["slices"]) for f in forms) + "};")
    L.append("template <int FORM, int SLICE, class M>")
    L.append("static __device__ __forceinline__ void body_slice(M& m, const Scalars& s, const int* pt) {")
    for fi, f in enumerate(forms):
        kw = "if" if fi == 0 else "else if"
        L.append(f"    {kw} constexpr (FORM == {fi}) body_{f}_slice<SLICE>(m, s, {args});")
    L.append("}")
    L.append("template <int FORM, class M>")
    L.append("static __device__ __forceinline__ void body(M& m, const Scalars& s, const int* pt) {")
    for fi, f in enumerate(forms):
        kw = "if" if fi == 0 else "else if"
        L.append(f"    {kw} constexpr (FORM == {fi}) body_{f}(m, s, {args});")
    L.append(f"    else if constexpr (FORM == 5) body_original_nvcc(m, s, {args});")
    L.append("}")
    L.append(f"}};  // struct {ns}")
    return "\n".join(L) + "\n", meta


NEST_FUNCS = {
    "jacobi7": ["jacobi7"],
    "swim": ["calc1", "calc2", "calc3"],
    "clover": ["ideal_gas", "pdv_predict", "advec_cell_x"],
    "wave4": ["wave4"],
    "d3q19": ["stream_collide"],
    "zsolve": ["z_solve_lhs"],
}


def generate_all(out_dir: str) -> dict:
    os.makedirs(out_dir, exist_ok=True)
    allmeta = {}
    for nest, fns in NEST_FUNCS.items():
        parts = ["// GENERATED by paper_2306_13002_b200/lowering.py from nests/" + nest +
                 ".c (original form) and paper_2306_13002_b200/emitted/" + nest + ".<variant>.c",
                 "// (host stage (a): this repo's optimizer, stage_a.py).  Do not edit: re-run `python -m "
                 "paper_2306_13002_b200.lowering`.",
                 "#pragma once", "namespace acs { namespace gen {"]
        for fn in fns:
            txt, meta = gen_function(nest, fn)
            parts.append(txt)
            allmeta[fn] = meta
            if nest == "wave4":
                txt, meta = gen_function(nest, fn, f32=True)
                parts.append(txt)
                allmeta[fn + "_f32"] = meta
        parts.append("}}  // namespace acs::gen")
        with open(os.path.join(out_dir, f"{nest}.cuh"), "w") as f:
            f.write("\n".join(parts) + "\n")
    return allmeta


if __name__ == "__main__":
    import json
    meta = generate_all(os.path.join(ROOT, "paper_2306_13002_b200", "csrc", "gen"))
    print(json.dumps(meta, indent=1))
