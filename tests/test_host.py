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


def test_scattered_set_is_independent_arrays_with_cached_pointer_tables():
    """allocate_scattered(shape) makes T independently allocated arrays per
    direction (memory.py:99-104); the pointer tables (one C loop) hold their
    data addresses and are rebuilt after the patch lists change."""
    s = fvb.BatchShape(2, 4, 3)
    sc = fvb.allocate_scattered(s)
    assert sc.in_block is None and len(sc.inputs) == 3
    tab = sc.input_table()
    assert tab.dtype == np.uint64
    assert [int(x) for x in tab] == [a.ctypes.data for a in sc.inputs]
    assert [int(x) for x in sc.output_table()] == [a.ctypes.data for a in sc.outputs]
    assert sc.input_table() is tab  # cached
    sc.inputs[1] = np.zeros(s.unknowns * s.haloed_cells)
    assert int(sc.input_table()[1]) == sc.inputs[1].ctypes.data
    c = sc.clone()
    assert all(a.ctypes.data != b.ctypes.data for a, b in zip(c.inputs, sc.inputs))
    assert all(a.tobytes() == b.tobytes() for a, b in zip(c.inputs, sc.inputs))


def test_scattered_set_shape_errors():
    s = fvb.BatchShape(2, 4, 3)
    sc = fvb.allocate_scattered(s)
    with pytest.raises(fvb.ShapeMismatchError):
        fvb.ScatteredPatchSet(s, sc.inputs[:2], sc.outputs)
    with pytest.raises(fvb.ShapeMismatchError):
        fvb.ScatteredPatchSet(s, [np.zeros(3)] * 3, sc.outputs)
    bad = fvb.ScatteredPatchSet(s, [np.zeros(144, dtype=np.float32)] * 3, sc.outputs)
    with pytest.raises(fvb.ShapeMismatchError):
        bad.input_table()  # float64 arrays only
    ro = np.zeros(64)
    ro.setflags(write=False)
    with pytest.raises(fvb.ShapeMismatchError):
        fvb.ScatteredPatchSet(s, sc.inputs, [ro] * 3).output_table()  # outputs must be writable


def test_host_accessibility_check_without_device():
    """fvb_host_accessible is a host lookup: plain numpy memory is not
    device-addressable until pinned / registered."""
    import ctypes

    from paper_2306_16731_b200 import _lib

    s = fvb.BatchShape(2, 4, 5)
    sc = fvb.allocate_scattered(s)
    bad = ctypes.c_int64()
    tab = sc.input_table()
    _lib.check(_lib.load().fvb_host_accessible(tab.ctypes.data, len(tab), 8 * 144, ctypes.byref(bad)))
    assert bad.value == 0


BATCH_FILES = [("2d_p3_t5_soa", 2, 3, 5, 7), ("3d_p2_t3_aosoa", 3, 2, 3, 8), ("2d_p4_t2_aos", 2, 4, 2, 9)]


def _to_soa(a, layout, n, t, m):
    if layout is fvb.Layout.AOS:
        return a.reshape(t, m, n).transpose(2, 0, 1).reshape(-1)
    if layout is fvb.Layout.AOSOA:
        return a.reshape(t, n, m).transpose(1, 0, 2).reshape(-1)
    return a


@pytest.mark.parametrize("name,d,p,t,seed", BATCH_FILES)
def test_batch_file_reads_reference_dumps_and_writes_them_back(name, d, p, t, seed, tmp_path):
    """Batch files written by the reference's dump_batch (oracle/gen_batchfile.py,
    patchdata.py:337-366): read_batch_file recovers the reference's input and
    golden output (= the pinned oracle's), write_batch_file reproduces the
    file byte for byte."""
    from golden_cases import GOLDEN
    from oracle import oracle
    from paper_2306_16731_b200.memory import read_batch_file, write_batch_file

    path = GOLDEN / f"batch_{name}.bin"
    shape, layout, inp, out = read_batch_file(path)
    assert shape == fvb.BatchShape(d, p, t) and layout.value == name.rsplit("_", 1)[1]
    q = oracle.init_field_soa(d, p, t, seed)
    ref_out, _ = oracle.step_c(d, p, t, q)
    n = d + 2
    assert _to_soa(inp, layout, n, t, (p + 2) ** d).tobytes() == q.tobytes()
    assert _to_soa(out, layout, n, t, p ** d).tobytes() == ref_out.tobytes()
    again = tmp_path / "again.bin"
    write_batch_file(again, shape, layout, inp, out)
    assert again.read_bytes() == path.read_bytes()


def test_batch_file_rejects_bad_headers_and_payloads(tmp_path):
    """load_batch's checks (patchdata.py:354-366): unknown count != d+2,
    truncated payload."""
    import struct

    from paper_2306_16731_b200.memory import read_batch_file

    bad = tmp_path / "bad.bin"
    bad.write_bytes(struct.pack("<5i", 2, 3, 5, 1, 1) + b"\0" * 8 * (5 * 25 + 5 * 9))
    with pytest.raises(ValueError, match="unknown count"):
        read_batch_file(bad)
    bad.write_bytes(struct.pack("<5i", 2, 3, 4, 1, 1) + b"\0" * 16)
    with pytest.raises(ValueError, match="payload"):
        read_batch_file(bad)
