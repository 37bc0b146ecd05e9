"""Host-side logic: shapes, enumerators, step plan, task DAG, user-function twins.

Mirrors the structure checks of the reference suite
(pkg/tests/test_patchdata.py, test_kernelgraph.py, test_equations.py)
against this package's host mirror.
"""

import itertools
import math

import numpy as np
import pytest

import paper_2306_16731_b200 as fvb
from paper_2306_16731_b200 import kernelgraph as kg
from paper_2306_16731_b200.patchdata import cell_linear, linear_offset
from golden_cases import records, small_arrays


def test_shape_validation_and_sizes():
    s = fvb.BatchShape(2, 16, 64)
    assert (s.unknowns, s.haloed_cells, s.interior_cells) == (4, 324, 256)
    assert s.input_size == 4 * 324 * 64 and s.output_size == 4 * 256 * 64
    for bad in ((1, 4, 1), (2, 1, 1), (3, 4, 0)):
        with pytest.raises(ValueError):
            fvb.BatchShape(*bad)


def test_enumerator_examples():
    # pkg/tests/test_patchdata.py:35-39
    s = fvb.BatchShape(2, 4, 1)
    assert linear_offset(fvb.Layout.AOS, s, True, 0, (-1, -1), 0) == 0
    assert linear_offset(fvb.Layout.AOS, s, True, 0, (0, -1), 1) == 5
    s2 = fvb.BatchShape(2, 4, 2)
    assert linear_offset(fvb.Layout.SOA, s2, True, 1, (-1, -1), 3) == 252


@pytest.mark.parametrize("layout", list(fvb.Layout))
@pytest.mark.parametrize("d,p,t", [(2, 3, 2), (3, 2, 3)])
def test_enumerator_bijective(layout, d, p, t):
    s = fvb.BatchShape(d, p, t)
    for haloed in (True, False):
        lo, hi = (-1, p + 1) if haloed else (0, p)
        seen = set()
        for patch in range(t):
            for cell in itertools.product(range(lo, hi), repeat=d):
                for k in range(d + 2):
                    seen.add(linear_offset(layout, s, haloed, patch, cell, k))
        m = p + 2 if haloed else p
        assert seen == set(range((d + 2) * m**d * t))


def test_cell_linear_coordinate_zero_fastest():
    s = fvb.BatchShape(3, 4, 1)
    assert cell_linear(s, True, (0, -1, -1)) == 1
    assert cell_linear(s, True, (-1, 0, -1)) == 6
    assert cell_linear(s, True, (-1, -1, 0)) == 36


def test_step_sequence_and_ranges():
    s = fvb.BatchShape(3, 4, 2)
    names = [k.name for k in kg.step_sequence(s, True)]
    assert names == ["copy", "flux_x", "flux_y", "flux_z", "lambda_x", "lambda_y", "lambda_z",
                     "acc_x", "acc_y", "acc_z", "reduce"]
    plan = fvb.build_plan(fvb.BatchShape(2, 16, 1), True)
    assert [st.range_size for st in plan.steps] == [256, 288, 288, 288, 288, 256, 256, 256]
    assert kg.invocations_per_patch(fvb.BatchShape(2, 4, 1), False) == 3 * 16 + 4 * 24
    assert kg.masked_per_patch(fvb.BatchShape(2, 4, 1), False) == 7 * 36 - (3 * 16 + 4 * 24)


def test_task_graph_structure():
    s = fvb.BatchShape(3, 4, 2)
    dag = fvb.build_task_graph(s, True)
    assert dag.node_count == 22
    order = kg.topological_order(dag)
    assert len(order) == dag.node_count
    # accumulate_n waits for copy, flux_n, lambda_n and acc_{n-1}; no cross-patch edges
    for u, v in dag.edges:
        assert u // 11 == v // 11
    pre = {}
    for u, v in dag.edges:
        pre.setdefault(v, set()).add(u % 11)
    assert pre[9 + 0] == {0, 3, 6, 8}  # acc_z <- copy, flux_z, lambda_z, acc_y
    assert pre[10] == {9}


def test_cycle_detection():
    s = fvb.BatchShape(2, 2, 1)
    dag = fvb.build_task_graph(s, False)
    dag.successors[6].append(0)
    dag.indegree[0] += 1
    with pytest.raises(fvb.GraphCycleError):
        kg.topological_order(dag)


def test_host_equations_match_reference_closure():
    p = fvb.EulerParameters()
    q = (1.3, 0.26, -0.39, 3.25)
    pr = (1.4 - 1.0) * (3.25 - (0.26 * 0.26 + -0.39 * -0.39) / (2.0 * 1.3))
    assert fvb.pressure(q, p) == pr
    un = 0.26 / 1.3
    assert fvb.flux(q, 0, p) == (0.26, 0.26 * un + pr, -0.39 * un, un * (3.25 + pr))
    assert fvb.max_eigenvalue(q, 1, p) == abs(-0.39 / 1.3) + math.sqrt(1.4 * pr / 1.3)
    with pytest.raises(fvb.InvalidStateError):
        fvb.pressure((-1.0, 0.0, 0.0, 1.0), p, check=True)
    with pytest.raises(ValueError):
        fvb.EulerParameters(1.0)
    assert not fvb.is_admissible((1.0, 0.0, 0.0, -1.0), p)


def test_context_validation_and_scale():
    with pytest.raises(ValueError):
        fvb.TimeStepContext(0.0, 0.1, fvb.EulerParameters())
    with pytest.raises(ValueError):
        fvb.TimeStepContext(1e-3, -1.0, fvb.EulerParameters())
    assert fvb.default_context().scale == 1e-3 / 0.1


def test_reduce_max_neutral_and_exact():
    assert fvb.reduce_max([]) == 0.0
    assert fvb.reduce_max([-1.0, -2.0]) == 0.0
    v = np.random.default_rng(0).uniform(0, 3, 1001)
    for strat in fvb.ReductionStrategy:
        assert fvb.reduce_max(v, strat) == float(v.max())


def test_scattered_set_views_contiguous_blocks():
    s = fvb.BatchShape(2, 4, 3)
    sc = fvb.allocate_scattered(s)
    sc.inputs[1][:] = 7.0
    assert (sc.in_block[144:288] == 7.0).all() and (sc.in_block[:144] == 0.0).all()
    with pytest.raises(fvb.ShapeMismatchError):
        fvb.ScatteredPatchSet(s, sc.inputs[:2], sc.outputs)
