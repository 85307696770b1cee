"""Parser for the satcc kernel subset (a small, independent re-implementation).

The grammar is the one the reference accepts (proj/src/parser.cpp:60-554,
proj/src/lexer.cpp:44-253): ``int``/``double`` only, statically dimensioned
arrays, ``void`` functions, ``#pragma`` lines, assignments (no compound ops in
printer output, but ``+= -= *= /=`` and ``++``/``--`` steps are desugared as the
reference does), ``if``/``else``, ``for``, blocks and calls to the 11 libm
builtins (proj/src/interp.cpp:74-91).

This module is used at BUILD time by ``lowering.py`` to turn the nest text —
the original source and the reference-emitted (accsat) form — into the
per-point device bodies of the sm_100a kernels, and by the host registry to
discover regions the way ``find_regions`` does (proj/src/ast.cpp:333-409).
It never executes a nest.
"""
from __future__ import annotations

import re
from dataclasses import dataclass, field
from typing import List, Optional

# ---------------------------------------------------------------------------
# Lexer

_TOKEN_RE = re.compile(r"""
    (?P<ws>[ \t\r\n]+)
  | (?P<lcomment>//[^\n]*)
  | (?P<bcomment>/\*.*?\*/)
  | (?P<float>(?:\d+\.\d*|\.\d+)(?:[eE][+-]?\d+)?[fF]?|\d+[eE][+-]?\d+[fF]?)
  | (?P<int>\d+)
  | (?P<ident>[A-Za-z_]\w*)
  | (?P<op>\+\+|--|\+=|-=|\*=|/=|<=|>=|==|!=|&&|\|\||[-+*/%<>=!(){}\[\];,])
""", re.VERBOSE | re.DOTALL)

KEYWORDS = {"int", "double", "void", "if", "else", "for"}


@dataclass
class Tok:
    kind: str   # 'int' 'float' 'ident' 'kw' 'op' 'pragma' 'end'
    text: str
    line: int
    pos: int = 0     # byte span in the source
    end: int = 0


def lex(src: str) -> List[Tok]:
    toks: List[Tok] = []
    pos = 0
    line = 1
    n = len(src)
    while pos < n:
        # pragma lines: captured byte-exact to end of line (with continuations)
        if src[pos] == "#":
            end = pos
            while True:
                nl = src.find("\n", end)
                if nl < 0:
                    nl = n
                if nl > 0 and src[nl - 1] == "\\" and nl < n:
                    end = nl + 1
                    continue
                break
            text = src[pos:nl]
            if not re.match(r"#\s*pragma\b", text):
                raise SyntaxError(f"{line}: only #pragma preprocessor lines are supported")
            toks.append(Tok("pragma", text, line, pos, nl))
            line += text.count("\n")
            pos = nl
            continue
        m = _TOKEN_RE.match(src, pos)
        if not m:
            raise SyntaxError(f"{line}: unexpected character {src[pos]!r}")
        kind = m.lastgroup
        text = m.group(kind)
        if kind in ("ws", "lcomment", "bcomment"):
            pass
        elif kind == "ident" and text in KEYWORDS:
            toks.append(Tok("kw", text, line, pos, m.end()))
        else:
            toks.append(Tok(kind, text, line, pos, m.end()))
        line += text.count("\n")
        pos = m.end()
    toks.append(Tok("end", "", line, n, n))
    return toks


# ---------------------------------------------------------------------------
# AST

@dataclass
class Expr:
    kind: str                 # int float var ref un bin call
    op: str = ""              # operator / callee / var name / array base
    kids: List["Expr"] = field(default_factory=list)
    text: str = ""            # literal spelling

    def __repr__(self):
        return print_expr(self)


@dataclass
class Stmt:
    kind: str                 # decl assign if for block call empty
    pragmas: List[str] = field(default_factory=list)
    # decl
    ty: str = ""
    names: List[tuple] = field(default_factory=list)   # (name, dims, init)
    # assign
    lhs: Optional[Expr] = None
    rhs: Optional[Expr] = None
    # if
    cond: Optional[Expr] = None
    then_s: Optional["Stmt"] = None
    else_s: Optional["Stmt"] = None
    # for
    init: Optional["Stmt"] = None
    step: Optional["Stmt"] = None
    body: Optional["Stmt"] = None
    loop_var: str = ""
    # block
    stmts: List["Stmt"] = field(default_factory=list)
    # call
    call: Optional[Expr] = None
    # byte span in the source, pragma lines included (beg, end)
    beg: int = -1
    end: int = -1


@dataclass
class Param:
    ty: str
    name: str
    dims: List[int]


@dataclass
class Function:
    name: str
    params: List[Param]
    body: Stmt


@dataclass
class Module:
    functions: List[Function]
    globals: List[Stmt]


# ---------------------------------------------------------------------------
# Parser

_BIN_PREC = [["||"], ["&&"], ["==", "!="], ["<", "<=", ">", ">="], ["+", "-"], ["*", "/", "%"]]


class _Parser:
    def __init__(self, toks: List[Tok]):
        self.t = toks
        self.p = 0

    def cur(self) -> Tok:
        return self.t[self.p]

    def adv(self) -> Tok:
        tok = self.t[self.p]
        self.p += 1
        return tok

    def check(self, text: str) -> bool:
        c = self.cur()
        return c.kind in ("op", "kw") and c.text == text

    def accept(self, text: str) -> bool:
        if self.check(text):
            self.p += 1
            return True
        return False

    def expect(self, text: str) -> Tok:
        if not self.check(text):
            c = self.cur()
            raise SyntaxError(f"{c.line}: expected {text!r}, got {c.text!r}")
        return self.adv()

    def ident(self) -> str:
        c = self.adv()
        if c.kind != "ident":
            raise SyntaxError(f"{c.line}: expected identifier, got {c.text!r}")
        return c.text

    def pragmas(self) -> List[str]:
        out = []
        while self.cur().kind == "pragma":
            out.append(self.adv().text)
        return out

    # -- module
    def module(self) -> Module:
        fns, globs = [], []
        while self.cur().kind != "end":
            prag = self.pragmas()
            if self.cur().kind == "end":
                break
            ty = self.adv().text
            if ty not in ("void", "int", "double"):
                raise SyntaxError(f"{self.cur().line}: expected declaration")
            name = self.ident()
            if self.check("("):
                params = self.params()
                body = self.block()
                fns.append(Function(name, params, body))
            else:
                self.p -= 1
                d = self.declarators(ty)
                d.pragmas = prag
                globs.append(d)
        return Module(fns, globs)

    def params(self) -> List[Param]:
        self.expect("(")
        out = []
        if self.accept(")"):
            return out
        if self.check("void") and self.t[self.p + 1].text == ")":
            self.adv()
            self.adv()
            return out
        while True:
            ty = self.adv().text
            name = self.ident()
            dims = []
            while self.accept("["):
                dims.append(int(self.adv().text))
                self.expect("]")
            out.append(Param(ty, name, dims))
            if not self.accept(","):
                break
        self.expect(")")
        return out

    def declarators(self, ty: str) -> Stmt:
        s = Stmt("decl", ty=ty)
        while True:
            name = self.ident()
            dims = []
            while self.accept("["):
                dims.append(int(self.adv().text))
                self.expect("]")
            init = self.expr() if self.accept("=") else None
            s.names.append((name, dims, init))
            if not self.accept(","):
                break
        self.expect(";")
        return s

    # -- statements
    def block(self) -> Stmt:
        self.expect("{")
        s = Stmt("block")
        while True:
            b0 = self.cur().pos
            prag = self.pragmas()
            if self.check("}"):
                if prag:
                    s.stmts.append(Stmt("empty", pragmas=prag))
                break
            st = self.stmt()
            st.pragmas = prag + st.pragmas
            if prag:
                st.beg = b0
            s.stmts.append(st)
        self.expect("}")
        return s

    def stmt(self) -> Stmt:
        b0 = self.cur().pos
        s = self._stmt()
        s.beg, s.end = b0, self.t[self.p - 1].end
        return s

    def _stmt(self) -> Stmt:
        prag = self.pragmas()
        c = self.cur()
        if c.kind == "op" and c.text == "{":
            s = self.block()
        elif c.kind == "kw" and c.text in ("int", "double"):
            self.adv()
            s = self.declarators(c.text)
        elif c.kind == "kw" and c.text == "if":
            self.adv()
            self.expect("(")
            cond = self.expr()
            self.expect(")")
            th = self.stmt()
            el = self.stmt() if self.accept("else") else None
            s = Stmt("if", cond=cond, then_s=th, else_s=el)
        elif c.kind == "kw" and c.text == "for":
            self.adv()
            self.expect("(")
            init = Stmt("empty") if self.check(";") else self.simple()
            self.expect(";")
            cond = None if self.check(";") else self.expr()
            self.expect(";")
            step = Stmt("empty") if self.check(")") else self.simple()
            self.expect(")")
            body = self.stmt()
            lv = init.lhs.op if init.kind == "assign" and init.lhs.kind == "var" else ""
            s = Stmt("for", init=init, cond=cond, step=step, body=body, loop_var=lv)
        elif c.kind == "op" and c.text == ";":
            self.adv()
            s = Stmt("empty")
        else:
            s = self.simple()
            self.expect(";")
        s.pragmas = prag + s.pragmas
        return s

    def simple(self) -> Stmt:
        """Assignment / compound assignment / ++ -- / call statement (no ';')."""
        lhs = self.postfix()
        for op in ("+=", "-=", "*=", "/="):
            if self.accept(op):
                rhs = self.expr()
                return Stmt("assign", lhs=lhs, rhs=Expr("bin", op[0], [lhs, rhs]))
        if self.accept("++"):
            return Stmt("assign", lhs=lhs, rhs=Expr("bin", "+", [lhs, Expr("int", text="1")]))
        if self.accept("--"):
            return Stmt("assign", lhs=lhs, rhs=Expr("bin", "-", [lhs, Expr("int", text="1")]))
        if self.accept("="):
            return Stmt("assign", lhs=lhs, rhs=self.expr())
        if lhs.kind == "call":
            return Stmt("call", call=lhs)
        raise SyntaxError(f"{self.cur().line}: expected assignment")

    # -- expressions
    def expr(self, level: int = 0) -> Expr:
        if level == len(_BIN_PREC):
            return self.unary()
        e = self.expr(level + 1)
        while self.cur().kind == "op" and self.cur().text in _BIN_PREC[level]:
            op = self.adv().text
            r = self.expr(level + 1)
            e = Expr("bin", op, [e, r])
        return e

    def unary(self) -> Expr:
        if self.accept("-"):
            return Expr("un", "-", [self.unary()])
        if self.accept("!"):
            return Expr("un", "!", [self.unary()])
        if self.accept("+"):
            return self.unary()
        return self.postfix()

    def postfix(self) -> Expr:
        c = self.adv()
        if c.kind == "int":
            return Expr("int", text=c.text)
        if c.kind == "float":
            return Expr("float", text=c.text)
        if c.kind == "op" and c.text == "(":
            e = self.expr()
            self.expect(")")
            return e
        if c.kind != "ident":
            raise SyntaxError(f"{c.line}: unexpected {c.text!r}")
        if self.accept("("):
            args = []
            if not self.accept(")"):
                while True:
                    args.append(self.expr())
                    if not self.accept(","):
                        break
                self.expect(")")
            return Expr("call", c.text, args)
        if self.check("["):
            idx = []
            while self.accept("["):
                idx.append(self.expr())
                self.expect("]")
            return Expr("ref", c.text, idx)
        return Expr("var", c.text)


def parse(src: str) -> Module:
    return _Parser(lex(src)).module()


# ---------------------------------------------------------------------------
# Printing (C syntax, minimal parentheses — same precedence table)

_PREC = {op: i for i, ops in enumerate(_BIN_PREC) for op in ops}


def print_expr(e: Expr, parent: int = -1) -> str:
    if e.kind in ("int", "float"):
        return e.text
    if e.kind == "var":
        return e.op
    if e.kind == "ref":
        return e.op + "".join(f"[{print_expr(k)}]" for k in e.kids)
    if e.kind == "call":
        return e.op + "(" + ", ".join(print_expr(k) for k in e.kids) + ")"
    if e.kind == "un":
        return e.op + print_expr(e.kids[0], 99)
    p = _PREC[e.op]
    s = print_expr(e.kids[0], p) + f" {e.op} " + print_expr(e.kids[1], p + 1)
    return f"({s})" if p < parent else s


# ---------------------------------------------------------------------------
# Regions (find_regions, proj/src/ast.cpp:333-398)

_MARKERS = re.compile(r"\b(gang|worker|vector|simd|teams|distribute|kernels|parallel)\b")


def is_marked(pragmas: List[str]) -> bool:
    """A loop is parallel-marked when one of its pragmas carries a marker
    (proj/src/ast.cpp:26-58: gang/worker/vector/parallel for/simd/teams/
    distribute/kernels/parallel)."""
    return any(_MARKERS.search(p) for p in pragmas)


@dataclass
class Region:
    function: Function
    index: int
    loops: List[Stmt]          # enclosing For stmts, outermost first; anchor last
    anchor: Stmt

    @property
    def marked_loops(self) -> List[Stmt]:
        return [l for l in self.loops if is_marked(l.pragmas)]


def find_regions(m: Module) -> List[Region]:
    """Deepest parallel-marked loops in source order (proj/src/ast.cpp:390-398)."""
    out: List[Region] = []

    def contains_marked(s: Stmt) -> bool:
        found = False

        def walk(t):
            nonlocal found
            if t is None or found:
                return
            if t.kind == "for" and is_marked(t.pragmas):
                found = True
                return
            for c in children(t):
                walk(c)
        for c in children(s):
            walk(c)
        return found

    def visit(s: Stmt, fn: Function, stack: List[Stmt]):
        if s is None:
            return
        if s.kind == "for":
            stack = stack + [s]
            if is_marked(s.pragmas) and not contains_marked(s):
                out.append(Region(fn, len(out), stack, s))
                return
        for c in children(s):
            visit(c, fn, stack)

    for fn in m.functions:
        visit(fn.body, fn, [])
    return out


def children(s: Stmt) -> List[Stmt]:
    out = []
    for c in (s.then_s, s.else_s, s.init, s.step, s.body):
        if c is not None:
            out.append(c)
    out.extend(s.stmts)
    return out
