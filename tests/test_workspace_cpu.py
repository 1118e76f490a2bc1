"""Session workspace planning (paper_2407_04991_b200/workspace.py).

* the forward's buffer plan: {ffn, q} and {h, attn} share storage, x is alone,
  check_plan accepts it, and padded layouts are never shared;
* check_plan rejects overlapping or undersized assignments (reference
  graphopt.py:333-346, test_graphopt.py:414-426);
* the planner restates the reference's: on random operator graphs built with the
  reference's own graph classes, ``analyze_lifetimes`` and first-fit
  ``plan_memory`` (definition order) give the reference's intervals, buffer
  sizes and assignment exactly (graphopt.py:265-330).
"""

import importlib
import os
import random
import sys

import pytest

from paper_2407_04991_b200 import workspace as W
from paper_2407_04991_b200.errors import PlanError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_forward_plan_shares_disjoint_buffers():
    plan = W.session_plan(rows=32, hidden=768, ffn=3072, ldk_h=768, ldk_f=3072, n_layers=12)
    a = plan.assignment
    assert a["q"] == a["ffn"] and a["h"] == a["attn"]
    assert len({a["x"], a["q"], a["h"]}) == 3
    assert plan.buffer_count == 3
    W.check_plan(plan)
    assert plan.peak_bytes == 32 * 2 * (3072 + 768 + 768)
    assert plan.peak_bytes < sum(plan.tensor_bytes.values())
    offs = plan.offsets()
    assert all(o % W.ALIGN == 0 for o in offs) and plan.arena_bytes() >= plan.peak_bytes


def test_padded_layouts_not_shared():
    plan = W.session_plan(rows=8, hidden=48, ffn=100, ldk_h=64, ldk_f=128, n_layers=2)
    assert len(set(plan.assignment.values())) == 5


def test_forward_lifetimes():
    ops = W.forward_ops(3)
    lt = W.analyze_lifetimes(ops)
    idx = {name: i for i, (name, _, _) in enumerate(ops)}
    assert lt["q"] == [(idx[f"qkv.{l}"], idx[f"attention.{l}"]) for l in range(3)]
    assert lt["ffn"] == [(idx[f"ffn1.{l}"], idx[f"ffn2.{l}"]) for l in range(3)]
    assert lt["attn"] == [(idx[f"attention.{l}"], idx[f"wo.{l}"]) for l in range(3)]
    with pytest.raises(PlanError):
        W.analyze_lifetimes([("a", ("x",), ())])


def test_check_plan_rejects_bad_plans():
    lt = {"a": [(0, 2)], "b": [(1, 3)], "c": [(4, 5)]}
    sizes = {"a": 10, "b": 10, "c": 20}
    plan = W.plan_memory(sizes, lt)
    W.check_plan(plan)
    assert plan.assignment["a"] != plan.assignment["b"]
    bad = W.ArenaPlan([20], {n: 0 for n in sizes}, sizes, lt)
    with pytest.raises(PlanError):
        W.check_plan(bad)
    small = W.ArenaPlan([10, 10, 10], {"a": 0, "b": 1, "c": 2}, sizes, lt)
    with pytest.raises(PlanError):
        W.check_plan(small)
    with pytest.raises(PlanError):
        W.plan_memory(sizes, lt, order="random")


def _reference_graphopt():
    sys.path.insert(0, ROOT)
    from oracle import ref_loader
    if not os.path.isdir(ref_loader.REF_SRC):
        pytest.skip("reference sources not available")
    ref_loader.load(with_pruning=False)
    return importlib.import_module(f"{ref_loader.PKG}.graphopt")


def _random_graph(go, rng: random.Random):
    """A random valid DAG of Gelu/Add nodes over the reference's graph classes
    (shapes vary so buffer sizes differ)."""
    from tinfer_ref.tensor import DType
    shapes = [(2, 2), (4, 4), (8, 2), (3, 5)]
    tensors = {"in0": go.TensorInfo("in0", (4, 4), DType.F32, "input")}
    nodes, live = [], ["in0"]
    n = rng.randint(3, 14)
    for i in range(n):
        out = f"t{i}" if i < n - 1 else "out"
        klass = "intermediate" if i < n - 1 else "output"
        tensors[out] = go.TensorInfo(out, rng.choice(shapes), DType.F32, klass)
        if len(live) >= 2 and rng.random() < 0.5:
            a, b = rng.sample(live, 2)
            nodes.append(go.Node(f"n{i}", "Add", [a, b], out))
        else:
            nodes.append(go.Node(f"n{i}", "Gelu", [rng.choice(live)], out))
        live.append(out)
    g = go.OpGraph(tensors, nodes)
    go.validate(g)
    return g


def test_planner_matches_reference_first_fit():
    go = _reference_graphopt()
    rng = random.Random(2407)
    for _ in range(200):
        g = _random_graph(go, rng)
        ref_lt = go.analyze_lifetimes(g)
        ref_plan = go.plan_memory(g, ref_lt)
        inter = {t for t, info in g.tensors.items() if info.klass == "intermediate"}
        ops = [(n.id, tuple(x for x in n.inputs if x in inter), (n.output,) if n.output in inter else ())
               for n in g.nodes]
        lt = W.analyze_lifetimes(ops)
        assert lt == {t: [iv] for t, iv in ref_lt.items()}
        plan = W.plan_memory({t: g.tensors[t].nbytes for t in lt}, lt, order="definition")
        W.check_plan(plan)
        assert plan.buffer_sizes == ref_plan.buffer_sizes
        assert plan.assignment == ref_plan.assignment


def test_graph_opt_cli_reports_the_forward_plan(tmp_path, capsys):
    """`tinfer graph-opt` prints what the reference's does (cli.py:163-180:
    nodes / launches / peak bytes, before -> after) for the fused forward, and
    writes the kernel sequence and buffer plan."""
    import json

    from paper_2407_04991_b200 import cli
    out = tmp_path / "plan.json"
    assert cli.main(["graph-opt", "--out", str(out)]) == 0
    text = capsys.readouterr().out
    assert "nodes:" in text and "launches:" in text and "peak bytes:" in text
    doc = json.loads(out.read_text())
    L = doc["config"]["num_layers"]
    assert len(doc["kernels"]) == 5 * L + 3  # decode step: LayerNorms folded into the GEMMs
    assert doc["assignment"]["q"] == doc["assignment"]["ffn"]
    assert cli.main(["graph-opt", "--tokens", "16"]) == 0
    assert f"-> {7 * L + 3}" in capsys.readouterr().out  # prefill: stand-alone LayerNorm kernels
    assert cli.main(["graph-opt", "--graph", "g.json"]) == 1
