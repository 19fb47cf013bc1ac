"""SAGA-NN front end and optimizer passes, CPU only."""

import pytest

import paper_1810_08403_b200 as sg
from paper_1810_08403_b200 import program as P
from paper_1810_08403_b200.errors import ProgramError


def test_gcn_program_fuses_to_gcn_kernel():
    q, reps = sg.optimize(sg.build_gcn(8, 4))
    assert q.fused.kind == "gcn"
    assert sg.validate_program(q) == []
    assert P.vertex_kind(q) == "W"


def test_ggcn_hoist_and_fuse():
    p = sg.build_ggcn(6, 3)
    assert P.matmul_rows(p.apply_edge, 30, 10) == 2 * 30          # 2|E| before
    q, rep = sg.hoist_vertex_computation(p)
    assert len(q.precompute) == 2 and sorted(s for s, _ in q.precompute.values()) == ["dest", "src"]
    assert P.matmul_rows(q.apply_edge, 30, 10, q.precompute) == 2 * 10   # 2|V| after
    assert not any(n.op == "matmul" for n in P.nodes(q.apply_edge))
    q2, rep2 = sg.fuse_sag(q)
    assert q2.fused.kind == "ggcn" and q2.fused.params == ("W_H", "W_C")


def test_hoist_idempotent():
    q, _ = sg.hoist_vertex_computation(sg.build_ggcn(5, 5))
    q2, rep = sg.hoist_vertex_computation(q)
    assert q2.apply_edge.key() == q.apply_edge.key() and rep.moved == []


def test_commnet_passthrough_unchanged_and_fused():
    p = sg.build_commnet(4, 4)
    q, rep = sg.hoist_vertex_computation(p)
    assert rep.moved == [] and q.apply_edge.key() == p.apply_edge.key()
    assert sg.fuse_sag(q)[0].fused.kind == "pass"


def test_mpgcn_matmul_blocks_fusion():
    p = sg.make_program(lambda e, p: P.sigmoid(e.src @ p.W_pool),
                        lambda v, acc, p: P.relu(acc @ p.W), "max",
                        {"W_pool": (4, 6), "W": (6, 3)}, 4, 3)
    q, rep = sg.fuse_sag(p)
    assert q.fused is None and rep.blocker == "matmul"


def test_scope_rules():  # accum is out of scope inside ApplyEdge
    with pytest.raises(sg.ProgramError):
        P.trace_udf(lambda e, p: P.Expr("input", name="accum", width=3), "edge", {}, 3)
    with pytest.raises(sg.ProgramError):
        P.trace_udf(lambda v, acc, p: P.Expr("input", name="edge.src", width=3), "vertex", {}, 3)


def test_validate_reports_width_mismatch():
    p = sg.make_program(lambda e, p: e.src, lambda v, acc, p: P.relu(acc @ p.W), "sum",
                        {"W": (16, 4)}, 8, 4, acc_width=16)
    diags = sg.validate_program(p)
    assert any("gather width 8" in d for d in diags)


def test_invalid_accumulator_and_dims():
    with pytest.raises(sg.ProgramError):
        sg.make_program(lambda e, p: e.src, lambda v, acc, p: acc, "mean", {}, 2, 2)
    with pytest.raises(sg.ProgramError):
        sg.build_gcn(0, 3)


def test_matmul_shape_error():
    with pytest.raises(sg.ProgramError):
        sg.make_program(lambda e, p: e.src @ p.W, lambda v, acc, p: acc, "sum", {"W": (5, 2)}, 3, 2)


def test_vertex_forms():
    assert P.vertex_form(sg.build_gcn(4, 3)) == ("w", "W")
    assert P.vertex_form(sg.build_commnet(4, 3)) == ("hc", "W_H", "W_C")
    swapped = sg.make_program(lambda e, p: e.src,
                              lambda v, acc, p: P.relu(acc @ p.B + v @ p.A), "sum",
                              {"A": (4, 3), "B": (4, 3)}, 4, 3)
    assert P.vertex_form(swapped) == ("hc", "A", "B")
    odd = sg.make_program(lambda e, p: e.src, lambda v, acc, p: P.sigmoid(acc @ p.W), "sum",
                          {"W": (4, 3)}, 4, 3)
    assert P.vertex_form(odd) is None


def test_reorder_linear_gather_pass():
    from paper_1810_08403_b200 import program as prog

    q, reps = prog.optimize(prog.build_gcn(602, 128), reorder=True)
    assert q.reorder and reps[-1].name == "reorder_linear_gather" and not reps[-1].blocker
    assert reps[-1].matmul_rows_after == "gather width 128"
    q, reps = prog.optimize(prog.build_gcn(16, 64), reorder=True)   # widening: keep the order
    assert not q.reorder and "f_out" in reps[-1].blocker
    q, reps = prog.optimize(prog.build_ggcn(64, 16), reorder=True)  # gated ApplyEdge: nonlinear
    assert not q.reorder and reps[-1].blocker
    q, reps = prog.optimize(prog.build_commnet(64, 16), reorder=True)  # ApplyVertex not ReLU(W accum)
    assert not q.reorder
    q, _ = prog.optimize(prog.build_gcn(602, 128))  # off by default
    assert not getattr(q, "reorder", False)


def test_ggnn_program_typed_hoist_and_gru():
    """GG-NN's edge stage is reduced to a per-type pre-computed scatter
    (A(type) (x) src hoisted per edge type); ApplyVertex is recognised as the GRU."""
    from paper_1810_08403_b200 import program as prog

    p = prog.build_ggnn(8, 3)
    assert prog.validate_program(p) == []
    q, (h, f) = prog.optimize(p)
    assert h.matmul_rows_before == "1*|E|" and h.matmul_rows_after == "0*|E| + 3*|V|"
    assert q.fused.kind == "typed" and q.fused.params == ("A",)
    assert prog.vertex_form(q) == ("gru", "W_z", "U_z", "W_r", "U_r", "W_h", "U_h")
    assert prog.matmul_rows(p.apply_edge, 100, 10) == 100
    assert prog.matmul_rows(q.apply_edge, 100, 10, q.precompute) == 30
    with pytest.raises(ProgramError):
        prog.build_ggnn(8, 0)
    with pytest.raises(ProgramError):   # the family is selected by edge.data only
        prog.make_program(lambda e, p: prog.typed_matmul(e.src, e.dest, p.A), lambda v, a, p: a, "sum",
                          {"A": (2, 4, 4)}, 4, 4)


def test_ggcn_fusion_requires_bare_vertex_matmuls():
    """a gate over non-bare hoisted sides (relu(src) @ W_H, (dest*dest) @ W_C)
    must not fuse as G-GCN (the kernel computes P = h W_H, Q = h W_C only)."""
    p = sg.make_program(
        lambda e, p: P.sigmoid(P.relu(e.src) @ p.W_H + (e.dest * e.dest) @ p.W_C) * e.src,
        lambda v, acc, p: P.relu(acc @ p.W), "sum",
        {"W_H": (4, 4), "W_C": (4, 4), "W": (4, 3)}, 4, 3)
    q, _ = sg.optimize(p)
    assert q.fused is None or q.fused.kind != "ggcn"
    from paper_1810_08403_b200.engine import lower_programs
    with pytest.raises(ProgramError):
        lower_programs([p])
    # the real G-GCN still fuses
    assert lower_programs([sg.build_ggcn(4, 3)])[0].kind == "ggcn"


def test_gru_apply_vertex_rejected_by_fused_executor():
    """ApplyEdge = e.src with a GRU ApplyVertex must raise, not run ReLU(accum W)."""
    from paper_1810_08403_b200.engine import lower_programs
    f = 4
    names = ["Wz", "Uz", "Wr", "Ur", "Wh", "Uh"]
    p = sg.make_program(lambda e, p: e.src,
                        lambda v, acc, p: P.gru(v, acc, *[getattr(p, n) for n in names]),
                        "sum", {n: (f, f) for n in names}, f, f)
    with pytest.raises(ProgramError, match="GRU"):
        lower_programs([p])
    assert [L.kind for L in lower_programs([sg.build_gcn(4, 3), sg.build_commnet(3, 3)])] == \
        ["gcn", "pass"]
