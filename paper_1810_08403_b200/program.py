"""SAGA-NN front end: UDF tracing, layer programs, optimizer passes, model zoo.

The SAGA-NN API of the reference SPEC: ``trace_udf`` / ``validate_program`` /
``evaluate_expr`` and ``LayerProgram`` (saga-frontend), the
two optimizer passes ``hoist_vertex_computation`` and ``fuse_sag``
 and the ``build_gcn`` / ``build_ggcn`` builders (model-zoo,
SPEC.md:521-550).  Users write the ApplyEdge UDF as ``apply_edge(edge, p)``
over ``edge.src / edge.dest / edge.data`` and the ApplyVertex UDF as
``apply_vertex(vertex, accum, p)``; Scatter and Gather are
not user-programmable, the accumulator is an enum.

``fuse_sag`` is where the kernel is chosen: a post-hoist ApplyEdge made only of
element-wise ops becomes a FusedGather descriptor naming the fused sm_100a
propagation mode that implements it.
"""

from dataclasses import dataclass, field

from .errors import ProgramError

ELEMENTWISE = {"add", "sub", "mul", "div", "max", "sigmoid", "tanh", "relu"}
EDGE_INPUTS = {"edge.src", "edge.dest", "edge.data"}
VERTEX_INPUTS = {"vertex", "accum"}


class Expr:
    """A node of a traced ExprGraph."""

    __slots__ = ("op", "args", "name", "width")

    def __init__(self, op, args=(), name=None, width=None):
        self.op, self.args, self.name, self.width = op, tuple(args), name, width

    # operator sugar -> traced nodes
    def __add__(self, o):
        return _bin("add", self, o)

    def __sub__(self, o):
        return _bin("sub", self, o)

    def __mul__(self, o):
        return _bin("mul", self, o)

    __rmul__ = __mul__

    def __truediv__(self, o):
        return _bin("div", self, o)

    def __matmul__(self, o):
        return matmul(self, o)

    def __repr__(self):
        if self.op in ("input", "param", "pre"):
            return self.name
        return f"{self.op}({', '.join(map(repr, self.args))})"

    def key(self):
        """Structural key (graph isomorphism for idempotence checks)."""
        if self.op in ("input", "param", "pre"):
            return (self.op, self.name)
        return (self.op,) + tuple(a.key() for a in self.args)


def _bin(op, a, b):
    if not isinstance(a, Expr) or not isinstance(b, Expr):
        raise ProgramError(f"'{op}' operands must be traced tensors")
    return Expr(op, (a, b), width=_bw(a, b, op))


def _bw(a, b, op):
    wa, wb = a.width, b.width
    if wa is None or wb is None:
        return wa if wb is None else wb
    if wa == wb or wb == 1:
        return wa
    if wa == 1:
        return wb
    raise ProgramError(f"'{op}' width mismatch {wa} vs {wb}")


def sigmoid(x):
    return Expr("sigmoid", (x,), width=x.width)


def tanh(x):
    return Expr("tanh", (x,), width=x.width)


def relu(x):
    return Expr("relu", (x,), width=x.width)


def maximum(a, b):
    return _bin("max", a, b)


def matmul(a, b):
    """Row convention x @ W (tensor.py:313).  ``W @ x`` (the paper's W (x) x) means the same."""
    if a.op == "param" and b.op != "param":
        a, b = b, a
    if b.op != "param" or not isinstance(b.width, tuple):
        raise ProgramError("matmul needs one per-row operand and one parameter matrix")
    rows, cols = b.width
    if a.width is not None and a.width != rows:
        raise ProgramError(f"matmul inner extents differ: {a.width} vs {rows}")
    return Expr("matmul", (a, b), width=cols)


def typed_matmul(x, labels, A):
    """GG-NN's A(edge.data) (x) edge.src (tensor.py:322-355 typed_matmul):
    row e times the parameter matrix A[labels[e]] of a (types, rows, cols) family."""
    if A.op != "param" or not isinstance(A.width, tuple) or len(A.width) != 3:
        raise ProgramError("typed_matmul needs a (types, rows, cols) parameter family")
    if labels.op != "input" or labels.name != "edge.data":
        raise ProgramError("typed_matmul selects its matrix by the integer edge label edge.data")
    _, rows, cols = A.width
    if x.width is not None and x.width != rows:
        raise ProgramError(f"typed_matmul inner extents differ: {x.width} vs {rows}")
    return Expr("typed_matmul", (x, labels, A), width=cols)


def gru(vertex, accum, Wz, Uz, Wr, Ur, Wh, Uh):
    """GRU(vertex, accum) ApplyVertex of GG-NN (Li et al.
    form, no biases): z = s(a Wz + h Uz), r = s(a Wr + h Ur), c = tanh(a Wh + (r*h) Uh),
    h' = (1 - z)*h + z*c."""
    ps = (Wz, Uz, Wr, Ur, Wh, Uh)
    for w in ps:
        if w.op != "param" or not isinstance(w.width, tuple) or len(w.width) != 2:
            raise ProgramError("gru needs six (F, F) parameter matrices")
    F = vertex.width
    if any(w.width != (F, F) for w in ps) or accum.width not in (None, F):
        raise ProgramError("gru state, input and parameter widths must all equal F")
    return Expr("gru", (vertex, accum) + ps, width=F)


class _Edge:
    def __init__(self, f_src, f_dest):
        self.src = Expr("input", name="edge.src", width=f_src)
        self.dest = Expr("input", name="edge.dest", width=f_dest)
        self.data = Expr("input", name="edge.data", width=1)


class _Params:
    def __init__(self, shapes):
        self._shapes = dict(shapes)

    def __getattr__(self, k):
        if k.startswith("_"):
            raise AttributeError(k)
        if k not in self._shapes:
            raise ProgramError(f"unknown parameter '{k}'")
        shape = tuple(self._shapes[k])
        # matrices keep their (rows, cols) (a typed family (types, rows, cols)); a bias
        # vector (n,) broadcasts like a row (b_lead)
        return Expr("param", name=k, width=shape if len(shape) >= 2 else shape[0])


def trace_udf(udf, kind, params, f_in):
    """Trace an ApplyEdge (kind='edge') or ApplyVertex (kind='vertex') UDF."""
    p = _Params(params)
    if kind == "edge":
        out = udf(_Edge(f_in, f_in), p)
        allowed = EDGE_INPUTS
    elif kind == "vertex":
        acc_w = params.get("__accum_width__", f_in)
        out = udf(Expr("input", name="vertex", width=f_in),
                  Expr("input", name="accum", width=acc_w), p)
        allowed = VERTEX_INPUTS
    else:
        raise ProgramError(f"unknown UDF kind '{kind}'")
    if not isinstance(out, Expr):
        raise ProgramError("a UDF must return a traced tensor")
    for n in inputs_of(out):
        if n not in allowed and not n.startswith("pre_"):
            raise ProgramError(f"placeholder '{n}' is out of scope in {kind} UDF")
    return out


def nodes(e):
    seen, out = set(), []

    def walk(x):
        if id(x) in seen:
            return
        seen.add(id(x))
        for a in x.args:
            walk(a)
        out.append(x)

    walk(e)
    return out


def inputs_of(e):
    return {n.name for n in nodes(e) if n.op in ("input", "pre")}


@dataclass
class FusedGather:
    """Fused-gather descriptor: which sm_100a propagation mode runs the SAG phase."""

    kind: str               # 'gcn' | 'pass' | 'ggcn' | 'generic'
    params: tuple = ()      # parameter names the fused kernel needs (ggcn: (W_H, W_C))


@dataclass
class PassReport:
    """SPEC.md:236-240."""

    name: str
    moved: list = field(default_factory=list)
    matmul_rows_before: str = ""
    matmul_rows_after: str = ""
    blocker: str = ""


@dataclass
class LayerProgram:
    """apply_edge / apply_vertex ExprGraphs, accumulator, named params."""

    apply_edge: Expr
    apply_vertex: Expr
    accumulator: str
    params: dict
    f_in: int
    f_out: int
    precompute: dict = field(default_factory=dict)  # name -> (side, Expr) hoisted per-vertex work
    fused: FusedGather = None


def make_program(apply_edge, apply_vertex, accumulator, params, f_in, f_out, acc_width=None):
    if accumulator not in ("sum", "max", "concat"):
        raise ProgramError(f"accumulator must be sum, max or concat (got '{accumulator}')")
    ae = trace_udf(apply_edge, "edge", params, f_in)
    av = trace_udf(apply_vertex, "vertex", dict(params, __accum_width__=acc_width or ae.width), f_in)
    return LayerProgram(ae, av, accumulator, dict(params), f_in, f_out)


def validate_program(p):
    """every violated rule as a diagnostic; [] means ok."""
    diags = []
    for n in inputs_of(p.apply_edge):
        if n not in EDGE_INPUTS and not n.startswith("pre_"):
            diags.append(f"apply_edge references out-of-scope placeholder '{n}'")
    for n in inputs_of(p.apply_vertex):
        if n not in VERTEX_INPUTS:
            diags.append(f"apply_vertex references out-of-scope placeholder '{n}'")
    if p.accumulator not in ("sum", "max", "concat"):
        diags.append(f"unknown accumulator '{p.accumulator}'")
    if p.accumulator == "concat":
        diags.append("concat accumulator requires deterministic order mode")
    acc_uses = [n for n in nodes(p.apply_vertex) if n.op == "input" and n.name == "accum"]
    ew = p.apply_edge.width
    for n in acc_uses:
        if n.width is not None and ew is not None and n.width != ew:
            diags.append(f"gather width {ew} feeds ApplyVertex expecting {n.width}")
    if p.apply_vertex.width not in (None, p.f_out):
        diags.append(f"apply_vertex output width {p.apply_vertex.width} != f_out {p.f_out}")
    return diags


def matmul_rows(e, n_edges, n_vertices, precompute=None):
    """Matmul row applications of one layer's ApplyEdge (tensor.py:133-158 counting)."""
    per_edge = sum(1 for n in nodes(e) if n.op in ("matmul", "typed_matmul"))
    per_vertex = sum(sum(1 if n.op == "matmul" else (n.args[1].width[0] if n.op == "typed_table" else 0)
                         for n in nodes(x)) for _, x in (precompute or {}).values())
    return per_edge * n_edges + per_vertex * n_vertices


def hoist_vertex_computation(p):
    """move maximal {src,params}- / {dest,params}-only subtrees
    containing a matmul out of ApplyEdge into per-vertex precompute."""
    pre = dict(p.precompute)
    moved = []

    def side_of(x):
        ins = inputs_of(x)
        if ins and ins <= {"edge.src"}:
            return "src"
        if ins and ins <= {"edge.dest"}:
            return "dest"
        return None

    def has_mm(x):
        return any(n.op in ("matmul", "typed_matmul") for n in nodes(x))

    def rewrite(x):
        if x.op == "typed_matmul" and side_of(x.args[0]) == "src":
            # per-type hoist: Y_t = vertex A_t for every type t per vertex,
            # the edge then selects Y_{edge.data}[src] -- a typed per-vertex scatter
            name = f"pre_src_typed{len(pre)}"
            vx = Expr("typed_table", (_to_vertex(x.args[0]), x.args[2]), width=x.width)
            pre[name] = ("src", vx)
            moved.append(f"{x!r} -> per-vertex per-type {name}")
            return Expr("select_type", (Expr("pre", name=name, width=x.width), x.args[1]),
                        width=x.width)
        s = side_of(x)
        if s is not None and has_mm(x):
            name = f"pre_{s}{len(pre)}"
            vx = _to_vertex(x)
            pre[name] = (s, vx)
            moved.append(f"{x!r} -> per-vertex {name}")
            return Expr("pre", name=name, width=x.width)
        if not x.args:
            return x
        return Expr(x.op, tuple(rewrite(a) for a in x.args), x.name, x.width)

    new_edge = rewrite(p.apply_edge)
    q = LayerProgram(new_edge, p.apply_vertex, p.accumulator, p.params, p.f_in, p.f_out, pre, p.fused)
    def per_vertex(v):
        return sum(1 if n.op == "matmul" else (n.args[1].width[0] if n.op == "typed_table" else 0)
                   for n in nodes(v))

    rep = PassReport("hoist_vertex_computation", moved,
                     f"{sum(1 for n in nodes(p.apply_edge) if n.op in ('matmul', 'typed_matmul'))}*|E|",
                     f"{sum(1 for n in nodes(new_edge) if n.op in ('matmul', 'typed_matmul'))}*|E| + "
                     f"{sum(per_vertex(v) for _, v in pre.values())}*|V|")
    return q, rep


def _to_vertex(x):
    if x.op == "input" and x.name in ("edge.src", "edge.dest"):
        return Expr("input", name="vertex", width=x.width)
    if not x.args:
        return x
    return Expr(x.op, tuple(_to_vertex(a) for a in x.args), x.name, x.width)


def _is(x, op, *names):
    return x.op == op and (not names or x.name in names)


def fuse_sag(p):
    """an element-wise-only (post-hoist) ApplyEdge becomes a FusedGather."""
    e = p.apply_edge
    mm = [n for n in nodes(e) if n.op in ("matmul", "typed_matmul")]
    if mm:
        rep = PassReport("fuse_sag", blocker="matmul")
        return LayerProgram(e, p.apply_vertex, p.accumulator, p.params, p.f_in, p.f_out,
                            p.precompute, None), rep
    kind, params = "generic", ()
    if p.accumulator == "max":
        if _is(e, "input", "edge.src"):
            kind = "max"
        elif e.op == "pre" and p.precompute[e.name][0] == "src":
            x = p.precompute[e.name][1]
            # sigmoid(vertex @ W_pool + b): MP-GCN's pooling edge network
            if x.op == "sigmoid" and x.args[0].op == "add":
                mm, bias = x.args[0].args
                if mm.op == "matmul" and _is(mm.args[0], "input", "vertex") and bias.op == "param":
                    kind, params = "max_pool", (mm.args[1].name, bias.name)
    if p.accumulator == "sum":
        if e.op == "select_type" and e.args[0].op == "pre" and p.precompute[e.args[0].name][0] == "src":
            kind = "typed"   # GG-NN: PASS gather over the per-type table (row src*T + type)
            params = (p.precompute[e.args[0].name][1].args[1].name,)
        elif _is(e, "input", "edge.src"):
            kind = "pass"
        elif e.op == "mul" and {a.name for a in e.args if a.op == "input"} == {"edge.src", "edge.data"}:
            kind = "gcn"
        elif e.op == "mul":
            a, b = e.args
            gate, other = (a, b) if a.op == "sigmoid" else (b, a)
            if gate.op == "sigmoid" and _is(other, "input", "edge.src") and gate.args[0].op == "add":
                x, y = gate.args[0].args
                sides = {}
                for t in (x, y):
                    if t.op == "pre":
                        sides[p.precompute[t.name][0]] = p.precompute[t.name][1]
                src_e, dst_e = sides.get("src"), sides.get("dest")
                # both hoisted sides must be the bare per-vertex matmul `vertex @ param`:
                # the kernel computes P = h W_H and Q = h W_C and nothing else
                def bare(t):
                    return t is not None and _is(t, "matmul") and \
                        _is(t.args[0], "input", "vertex") and t.args[1].op == "param"

                if bare(src_e) and bare(dst_e) and x.op == "pre" and y.op == "pre" and \
                        p.precompute[x.name][0] == "src":
                    kind = "ggcn"
                    params = (src_e.args[1].name, dst_e.args[1].name)
    fg = FusedGather(kind, params)
    rep = PassReport("fuse_sag", [f"SAG -> FusedGather({kind})"])
    return LayerProgram(e, p.apply_vertex, p.accumulator, p.params, p.f_in, p.f_out,
                        p.precompute, fg), rep


def evaluate_expr(e, bindings):
    """evaluate a traced graph on CUDA tensors with the libsagann ops.

    ``bindings`` maps input/param/pre names ('edge.src', 'edge.data', 'W', ...) to tensors;
    row-wise semantics follow the reference primitives (tensor.py:204-319)."""
    from . import ops

    memo = {}

    def ev(x):
        if id(x) in memo:
            return memo[id(x)]
        if x.op in ("input", "param", "pre"):
            if x.name not in bindings:
                raise ProgramError(f"missing binding for '{x.name}'")
            v = bindings[x.name]
        elif x.op == "matmul":
            v = ops.matmul(ev(x.args[0]), ev(x.args[1]))
        elif x.op in ("sigmoid", "tanh", "relu"):
            v = getattr(ops, x.op)(ev(x.args[0]))
        else:
            v = ops.elementwise(x.op, ev(x.args[0]), ev(x.args[1]))
        memo[id(x)] = v
        return v

    return ev(e)


def optimize(p, reorder=False):
    """hoist then fuse (the paper's pipeline); optionally then
    ``reorder_linear_gather``."""
    q, r1 = hoist_vertex_computation(p)
    q, r2 = fuse_sag(q)
    if not reorder:
        return q, [r1, r2]
    q, r3 = reorder_linear_gather(q)
    return q, [r1, r2, r3]


def reorder_linear_gather(p):
    """Move ApplyVertex's weight in front of the Gather when that narrows the propagation.

    For a fused sum gather whose ApplyEdge is linear in edge.src (GCN: src * edge.data;
    passthrough) and ApplyVertex = ReLU(W (x) accum):
        ReLU((sum_e w_e h[src_e]) W) == ReLU(sum_e w_e (h W)[src_e])
    so the layer can run Y = h W per vertex (a GEMM) and propagate Y at width f_out
    instead of h at width f_in -- the same function, re-associated: results agree with
    the reference order to fp32 rounding, not bitwise (the aggregate a = A h is never
    formed).  Applied only when f_out < f_in (the propagation is the dominant cost,
    SURVEY.md §8(d)).  Sets ``p.reorder`` (an attribute the executor reads)."""
    ok = (p.fused is not None and p.fused.kind in ("gcn", "pass") and p.accumulator == "sum"
          and vertex_kind(p) is not None)
    q = LayerProgram(p.apply_edge, p.apply_vertex, p.accumulator, p.params, p.f_in, p.f_out,
                     p.precompute, p.fused)
    if not ok:
        q.reorder = False
        return q, PassReport("reorder_linear_gather", blocker="not a linear sum gather + ReLU(W accum)")
    if p.f_out >= p.f_in:
        q.reorder = False
        return q, PassReport("reorder_linear_gather", blocker=f"f_out {p.f_out} >= f_in {p.f_in}")
    q.reorder = True
    return q, PassReport("reorder_linear_gather", [f"{vertex_kind(p)} before Gather"],
                         matmul_rows_before=f"gather width {p.f_in}",
                         matmul_rows_after=f"gather width {p.f_out}")


def vertex_kind(p):
    """Recognise ApplyVertex = ReLU(W (x) accum); returns the W param name."""
    v = p.apply_vertex
    if v.op == "relu" and v.args[0].op == "matmul":
        x, W = v.args[0].args
        if _is(x, "input", "accum") and W.op == "param":
            return W.name
    return None


def vertex_form(p):
    """The ApplyVertex forms the executor lowers onto GEMMs:
    ('w', W)         ReLU(W (x) accum)                    GCN / G-GCN / MP-GCN
    ('hc', W_H, W_C) ReLU(W_H (x) vertex + W_C (x) accum) CommNet
    or None."""
    W = vertex_kind(p)
    if W is not None:
        return ("w", W)
    v = p.apply_vertex
    if v.op == "gru" and _is(v.args[0], "input", "vertex") and _is(v.args[1], "input", "accum"):
        return ("gru",) + tuple(w.name for w in v.args[2:])
    if v.op == "relu" and v.args[0].op == "add":
        def mm(t, name):
            if t.op == "matmul" and _is(t.args[0], "input", name) and t.args[1].op == "param":
                return t.args[1].name
            return None

        a, b = v.args[0].args
        wh, wc = mm(a, "vertex"), mm(b, "accum")
        if wh is None or wc is None:
            wh, wc = mm(b, "vertex"), mm(a, "accum")
        if wh is not None and wc is not None:
            return ("hc", wh, wc)
    return None


# ------------------------------------------------------------------ model zoo
def build_gcn(f_in, f_out):
    """GCN: ApplyEdge = src x edge.data, sum, ReLU(W accum)."""
    if f_in < 1 or f_out < 1:
        raise ProgramError("invalid dimensions")
    return make_program(lambda e, p: e.src * e.data,
                        lambda v, acc, p: relu(matmul(acc, p.W)),
                        "sum", {"W": (f_in, f_out)}, f_in, f_out)


def build_ggcn(f_in, f_out):
    """G-GCN (listing :172-173 -- W_H on src, W_C on dest, Appendix B.1)."""
    if f_in < 1 or f_out < 1:
        raise ProgramError("invalid dimensions")
    return make_program(
        lambda e, p: sigmoid(matmul(e.src, p.W_H) + matmul(e.dest, p.W_C)) * e.src,
        lambda v, acc, p: relu(matmul(acc, p.W)),
        "sum", {"W_H": (f_in, f_in), "W_C": (f_in, f_in), "W": (f_in, f_out)}, f_in, f_out)


def build_commnet(f_in, f_out):
    """CommNet: ApplyEdge = edge.src (no edge-parallel compute), sum,
    ApplyVertex = ReLU(W_H (x) vertex + W_C (x) accum); params p = [W_H, W_C]."""
    if f_in < 1 or f_out < 1:
        raise ProgramError("invalid dimensions")
    return make_program(lambda e, p: e.src,
                        lambda v, acc, p: relu(matmul(v, p.W_H) + matmul(acc, p.W_C)), "sum",
                        {"W_H": (f_in, f_out), "W_C": (f_in, f_out)}, f_in, f_out)


def build_mpgcn(f_in, f_pool, f_out):
    """MP-GCN: ApplyEdge = sigmoid(W_pool src + b), Gather.accumulator =
    max, ApplyVertex = ReLU(W accum).  The edge network depends on src only, so the hoist
    pass moves it to one per-vertex GEMM and the SAG phase becomes a fused max gather."""
    if min(f_in, f_pool, f_out) < 1:
        raise ProgramError("invalid dimensions")
    return make_program(lambda e, p: sigmoid(matmul(e.src, p.W_pool) + p.b),
                        lambda v, acc, p: relu(matmul(acc, p.W)), "max",
                        {"W_pool": (f_in, f_pool), "b": (f_pool,), "W": (f_pool, f_out)},
                        f_in, f_out, acc_width=f_pool)


def build_ggnn(f, edge_types):
    """GG-NN: ApplyEdge = A(edge.data) (x) edge.src with
    one (f, f) matrix per edge type, Gather(sum), ApplyVertex = GRU(vertex, accum)."""
    if f < 1 or edge_types < 1:
        raise ProgramError("invalid dimensions")
    shapes = {"A": (edge_types, f, f)}
    shapes.update({k: (f, f) for k in ("W_z", "U_z", "W_r", "U_r", "W_h", "U_h")})
    return make_program(lambda e, p: typed_matmul(e.src, e.data, p.A),
                        lambda v, acc, p: gru(v, acc, p.W_z, p.U_z, p.W_r, p.U_r, p.W_h, p.U_h),
                        "sum", shapes, f, f)


MODELS = {"gcn": build_gcn, "ggcn": build_ggcn, "commnet": build_commnet, "mpgcn": build_mpgcn,
          "ggnn": build_ggnn}
