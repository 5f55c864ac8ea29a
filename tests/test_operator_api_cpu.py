"""Host-side operator vocabulary, replayed from the reference's own tests.

Planners over explicit scans (reference tests/test_load_balance.py), the AUTO
heuristic, the frontier containers (tests/test_frontier.py) and the INEXACT
culling oracle pinned to golden vectors made by running the reference
(oracle/make_cull_golden.py).  No GPU needed.
"""
from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from paper_1701_01170_b200 import (CooGraph, Frontier, FrontierPair, LbParams, Strategy,
                                   choose_strategy, coo_to_csr, plan_lb_input, plan_lb_output,
                                   plan_pairs, plan_thread_expand, plan_twc)
from paper_1701_01170_b200.load_balance import build_plan, scan_from_degrees

GOLDEN = Path(__file__).parent / "golden"


def frontier_of(*items):
    return Frontier.from_items(np.array(items, dtype=np.int64))


def scan_of(*degrees):
    return scan_from_degrees(np.array(degrees, dtype=np.int64))[0]


def nested_loop_pairs(scan):
    """Every (input item, output slot) pair by definition (reference _oracles.py:159-166)."""
    return np.array([(i, s) for i in range(len(scan) - 1)
                     for s in range(int(scan[i]), int(scan[i + 1]))], dtype=np.int64).reshape(-1, 2)


# test_load_balance.py:35-50
def test_prefix_sum():
    scan = scan_of(3, 1, 1, 1)
    assert scan.tolist() == [0, 3, 4, 5, 6]


# test_load_balance.py:53-72
def test_thread_expand():
    scan = scan_of(3, 1, 1, 1)
    assert plan_thread_expand(frontier_of(9, 9, 9, 9), scan).num_chunks == 4
    plan = plan_thread_expand(frontier_of(5, 6, 7), scan_of(2, 0, 1))
    assert plan.num_chunks == 3 and plan.chunks[1].slot_begin == plan.chunks[1].slot_end == 2
    plan = plan_thread_expand(frontier_of(1, 2, 3, 4), scan)
    for i, ch in enumerate(plan.chunks):
        assert (ch.slot_begin, ch.slot_end) == (int(scan[i]), int(scan[i + 1]))


# test_load_balance.py:75-108
def test_twc_classes_and_order():
    plan = plan_twc(frontier_of(0, 1, 2), scan_of(500, 40, 3), small_cut=32, large_cut=256)
    assert [c.size_class for c in plan.chunks] == ["large", "medium", "small"]
    plan = plan_twc(frontier_of(0, 1, 2), scan_of(256, 32, 31), small_cut=32, large_cut=256)
    assert {c.item_begin: c.size_class for c in plan.chunks} == {0: "large", 1: "medium",
                                                                  2: "small"}
    plan = plan_twc(frontier_of(*range(5)), scan_of(1, 300, 40, 2, 500), small_cut=32,
                    large_cut=256)
    assert [c.size_class for c in plan.chunks] == ["large", "large", "medium", "small", "small"]
    assert [c.item_begin for c in plan.chunks] == [1, 4, 2, 0, 3]
    f = frontier_of(0, 1, 2)
    twc, te = plan_twc(f, scan_of(3, 1, 2)), plan_thread_expand(f, scan_of(3, 1, 2))
    assert [(c.slot_begin, c.slot_end, c.item_begin) for c in twc.chunks] == \
        [(c.slot_begin, c.slot_end, c.item_begin) for c in te.chunks]
    with pytest.raises(ValueError):
        plan_twc(f, scan_of(3, 1, 2), small_cut=8, large_cut=8)


# test_load_balance.py:111-139
def test_lb_output():
    plan = plan_lb_output(scan_of(4, 4, 2), 10, chunk_size=4)
    assert [(c.slot_begin, c.slot_end) for c in plan.chunks] == [(0, 4), (4, 8), (8, 10)]
    lut = {int(s): int(i) for i, s in plan_pairs(plan_lb_output(scan_of(3, 1, 1, 1), 6, 4))}
    assert lut[3] == 1
    plan = plan_lb_output(scan_of(10), 10, chunk_size=4)
    assert plan.num_chunks == 3 and all(c.item_begin == 0 for c in plan.chunks)
    rng = np.random.default_rng(1)
    for _ in range(50):
        degs = rng.integers(0, 20, size=rng.integers(0, 30))
        scan, total = scan_from_degrees(degs)
        n = int(rng.integers(1, 9))
        assert plan_lb_output(scan, total, chunk_size=n).num_chunks == -(-total // n)
    with pytest.raises(ValueError):
        plan_lb_output(scan_of(1), 1, chunk_size=0)


# test_load_balance.py:142-157
def test_lb_input():
    plan = plan_lb_input(Frontier.from_items(np.zeros(8, dtype=np.int64)), scan_of(*([1] * 8)), 4)
    assert plan.num_chunks == 2
    scan = scan_of(2, 3, 0, 5)
    ch = plan_lb_input(Frontier.from_items(np.zeros(4, dtype=np.int64)), scan, 2).chunks[1]
    assert ch.slot_begin == int(scan[2]) and ch.slot_end == int(scan[4])
    assert plan_lb_input(frontier_of(), scan_of(), 4).num_chunks == 0


# test_load_balance.py:160-198: choose_strategy(g, f) takes the Frontier
def _graph_with(n, m):
    src = np.arange(m, dtype=np.int64) % n
    dst = (np.arange(m, dtype=np.int64) * 7 + 1) % n
    return coo_to_csr(CooGraph(n, src, dst), dedup=False)


def test_choose_strategy():
    g = _graph_with(1000, 8000)
    assert choose_strategy(g, Frontier.from_items(np.zeros(100, dtype=np.int64))) == \
        Strategy.LB_LIGHT
    assert choose_strategy(g, Frontier.from_items(np.zeros(10000, dtype=np.int64))) == Strategy.LB
    assert choose_strategy(_graph_with(1000, 2000), frontier_of(0)) == Strategy.TWC
    f = Frontier.from_items(np.zeros(10, dtype=np.int64))
    assert choose_strategy(_graph_with(1000, 4999), f) == Strategy.TWC
    assert choose_strategy(_graph_with(1000, 5000), f) == Strategy.LB_LIGHT
    assert choose_strategy(g, Frontier.from_items(np.zeros(4095, dtype=np.int64))) == \
        Strategy.LB_LIGHT
    assert choose_strategy(g, Frontier.from_items(np.zeros(4096, dtype=np.int64))) == Strategy.LB


# test_load_balance.py:201-221 (plans tile the work exactly once), over
# explicit scans so no device scan is needed
@pytest.mark.parametrize("strategy", [Strategy.THREAD_EXPAND, Strategy.TWC, Strategy.LB,
                                      Strategy.LB_LIGHT, Strategy.LB_CULL])
def test_plans_tile_work_exactly(strategy):
    rng = np.random.default_rng(abs(hash(strategy.value)) % 2**32)
    params = LbParams(small_cut=4, large_cut=16, chunk_size=8, items_per_chunk=4)
    g = _graph_with(64, 512)
    for _ in range(25):
        degs = rng.integers(0, 40, size=int(rng.integers(0, 60)))
        scan, total = scan_from_degrees(degs)
        f = Frontier.from_items(np.zeros(len(degs), dtype=np.int64))
        plan = build_plan(g, f, strategy, params, scan=scan, total=total)
        got = plan_pairs(plan)
        got = got[np.lexsort((got[:, 1], got[:, 0]))]
        assert np.array_equal(got, nested_loop_pairs(scan))


# tests/test_frontier.py:37-77 (host contract of the device-backed Frontier)
def test_frontier_pair_and_buffer():
    pair = FrontierPair.create()
    pair.input.set_items([1])
    pair.output.set_items([2])
    pair.swap()
    assert pair.input.to_array().tolist() == [2] and len(pair.output) == 0
    a, b = pair.input, pair.output
    pair.swap()
    pair.swap()
    assert pair.input is a and pair.output is b
    f = Frontier()
    f.set_items(np.arange(10))
    cap = f.capacity
    f.set_items(np.arange(cap + 1))
    assert f.capacity >= 2 * cap
    src = np.arange(4, dtype=np.int64)
    f.set_items(src)
    src[0] = 99
    assert f.to_array()[0] == 0


def test_inexact_cull_oracle_matches_reference_golden():
    """oracle cull_inexact == the reference's _apply_culling outputs, exactly."""
    from oracle import graphfx_port as port

    z = np.load(GOLDEN / "cull_inexact.npz")
    for k in range(int(z["count"])):
        bm, team, local, bb, lb, dom = z[f"cfg_{k}"].tolist()
        got = port.cull_inexact(z[f"items_{k}"], bool(bm), team, local, bb, lb, dom)
        assert np.array_equal(got, z[f"out_{k}"]), k
