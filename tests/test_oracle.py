"""Pin the CPU oracle (oracle/) to the reference before trusting it.

Checks every restatement against the fixtures the reference itself produced
(tests/golden, oracle/gen_golden.py), SURVEY.md Appendix B's SHA-256 table and
the reference's frozen LCG KAT (pkg/tests/test_bench.py:46-69).
"""

import hashlib

import numpy as np
import pytest

from golden_cases import APPENDIX_B, case_input_soa, records, small_arrays
from oracle import oracle


def _sha(arr):
    return hashlib.sha256(np.ascontiguousarray(arr, dtype="<f8").tobytes()).hexdigest()


def test_lcg_first_cell_kat():
    # pkg/tests/test_bench.py:46-69 frozen values for seed 0, d=2
    q = oracle.init_field_soa(2, 4, 1, 0)
    M = 36
    assert q[0] == 0.6173129823174408
    assert q[M] == -0.24587652614192054
    assert q[2 * M] == 0.06501745439736487
    assert q[3 * M] == 2.8069511536083835


def test_lcg_jump_matches_sequential_draws():
    s = 12345
    seq = s
    for i in range(1, 200):
        seq = (seq * oracle.LCG_A + oracle.LCG_C) & oracle.MASK64
        assert oracle.lcg_jump(s, i) == seq
        assert oracle.lib().fvo_lcg_jump(s, i) == seq


@pytest.mark.parametrize("d,p,t,seed", [(2, 4, 3, 5), (3, 3, 2, 99), (2, 7, 2, 1 << 63)])
def test_c_field_matches_python_field(d, p, t, seed):
    a = oracle.init_field_soa(d, p, t, seed)
    b = oracle.init_field_python(d, p, t, seed)
    assert a.tobytes() == b.tobytes()


def test_shard_field_equals_whole_field():
    d, p, t = 2, 5, 9
    whole = oracle.init_field_soa(d, p, t, 3)
    n, M, _ = oracle.sizes(d, p, t)
    part = np.zeros_like(whole)
    lib = oracle.lib()
    lib.fvo_init_field_soa(d, p, t, 3, 1.4, part.ctypes.data, 0, 4, 1)
    lib.fvo_init_field_soa(d, p, t, 3, 1.4, part.ctypes.data, 4, 5, 2)
    assert part.tobytes() == whole.tobytes()


@pytest.mark.parametrize("key", sorted(APPENDIX_B))
def test_appendix_b_golden_table(key):
    d, p, t, seed = key
    reduced, sha_in, sha_out = APPENDIX_B[key]
    q = oracle.init_field_soa(d, p, t, seed)
    assert _sha(oracle.soa_to_aos_patches(q, d, p, t, True))[:16] == sha_in
    out, red = oracle.step_c(d, p, t, q)
    assert repr(red) == reduced
    assert _sha(oracle.soa_to_aos_patches(out, d, p, t, False))[:16] == sha_out


@pytest.mark.parametrize("rec", records(), ids=lambda r: r["name"])
def test_oracles_match_reference_fixtures(rec):
    d, p, t = rec["d"], rec["p"], rec["t"]
    q = case_input_soa(rec, oracle)
    assert _sha(oracle.soa_to_aos_patches(q, d, p, t, True)) == rec["sha256_in"]
    kw = dict(dt=rec["dt"], h=rec["h"], gamma=rec["gamma"], with_reduction=rec["with_reduction"])
    out_c, red_c = oracle.step_c(d, p, t, q, **kw)
    assert _sha(oracle.soa_to_aos_patches(out_c, d, p, t, False)) == rec["sha256_out"]
    if rec["with_reduction"]:
        assert red_c.hex() == rec["reduced_hex"]
    else:
        assert red_c is None
    if out_c.size <= 300_000:
        out_n, red_n = oracle.step_numpy(d, p, t, q, **kw)
        assert out_n.tobytes() == out_c.tobytes()
        assert red_n == red_c


def test_small_case_arrays_elementwise():
    z = small_arrays()
    by_name = {r["name"]: r for r in records()}
    names = sorted({k.split("/")[0] for k in z.files})
    assert len(names) >= 20
    for name in names:
        rec = by_name[name]
        d, p, t = rec["d"], rec["p"], rec["t"]
        q = oracle.aos_patches_to_soa(z[name + "/in"], d, p, t, True)
        out, _ = oracle.step_c(d, p, t, q, dt=rec["dt"], h=rec["h"], gamma=rec["gamma"],
                               with_reduction=rec["with_reduction"])
        np.testing.assert_array_equal(oracle.soa_to_aos_patches(out, d, p, t, False),
                                      z[name + "/out"])


def test_threads_do_not_change_bits():
    q = oracle.init_field_soa(3, 4, 7, 21)
    a = oracle.step_c(3, 4, 7, q, threads=1, lam_patch=True)
    b = oracle.step_c(3, 4, 7, q, threads=3, lam_patch=True)
    assert a[0].tobytes() == b[0].tobytes() and a[1] == b[1]
    assert a[2].tobytes() == b[2].tobytes()
    assert a[1] == a[2].max()


def test_halo_refresh_restatement_periodic_identity():
    """A field built as a global periodic function: the refreshed halo of
    every patch must equal the global field sampled one cell outside."""
    d, p, grid = 2, 3, (3, 2)
    n, t = 4, 6
    gx, gy = grid[0] * p, grid[1] * p
    field = np.arange(n * gx * gy, dtype=np.float64).reshape(n, gy, gx)
    interior = np.empty((n, t, p * p))
    for patch in range(t):
        ix, iy = patch % 3, patch // 3
        interior[:, patch] = field[:, iy * p:(iy + 1) * p, ix * p:(ix + 1) * p].reshape(n, -1)
    halo = oracle.refresh_halos_soa(d, p, grid, interior.reshape(-1)).reshape(n, t, p + 2, p + 2)
    for patch in range(t):
        ix, iy = patch % 3, patch // 3
        for cy in range(-1, p + 1):
            for cx in range(-1, p + 1):
                gxx, gyy = (ix * p + cx) % gx, (iy * p + cy) % gy
                assert np.array_equal(halo[:, patch, cy + 1, cx + 1], field[:, gyy, gxx])
