"""Layer-wise tuning API (backends::tune_with_report, reference
backends.cpp:73-176 and test_backends.cpp's injected-cost cases) on CPU: the
injected cost model assigns every compute node of the three role graphs,
reports node-major records, and rejects a cost table that misses a node."""
import json

import pytest

import paper_2205_10357_b200 as P
from paper_2205_10357_b200 import workloads as W


def _members(m):
    names = {}
    for role in ("inference", "train_fwd", "train_bwd"):
        for g in m.describe[role]["groups"]:
            for mbr in g["members"]:
                names[mbr] = g["backend"]
    return names


def test_injected_costs_assign_every_node_without_a_device():
    m = P.CompiledModel(W.c1_small_cnn(4, bn=True))
    names = _members(m)
    rep = m.tune(injected={n: {b: float(i + 1)} for i, (n, b) in enumerate(sorted(names.items()))})
    for role in ("inference", "train_fwd", "train_bwd"):
        recs = rep[role]["records"]
        assert recs and all(r["chosen"] for r in recs)          # one supporting backend per op
        assert {r["node"] for r in recs} <= set(names)
        assert all(r["backend"] == names[r["node"]] for r in recs)
        assert "cost_us" in rep[role]["text"]
    assert rep["attached_launches"] == 0                          # injected: no tile choices


def test_injected_cost_table_must_be_total():
    m = P.CompiledModel(W.c1_small_cnn(4, bn=False))
    names = _members(m)
    first = sorted(names)[0]
    with pytest.raises(P.NNCError) as e:
        m.tune(injected={n: {b: 1.0} for n, b in names.items() if n != first})
    assert e.value.code == "BadDocument" and first in str(e.value)


def test_plans_carry_a_tile_field():
    m = P.CompiledModel(W.c1_small_cnn(4, bn=False))
    for role in ("inference", "train_fwd", "train_bwd"):
        for g in m.describe[role]["groups"]:
            for L in g["launches"]:
                assert L["tile"] == 0
