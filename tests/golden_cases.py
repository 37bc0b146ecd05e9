"""Loader for the committed golden fixtures (tests/golden/, made by
oracle/gen_golden.py from the reference itself)."""

import json
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"

# (d, p, T, seed) -> (reduced, sha256(in)[:16], sha256(out)[:16])
APPENDIX_B = {
    (2, 4, 1, 240): ("2.2702036798319316", "35dc49adc6c51089", "6524cdd7aa92c4e3"),
    (2, 4, 4, 240): ("2.3260398813009844", "6c9c3bf66c6c137c", "a81635f44a05c035"),
    (2, 4, 16, 240): ("2.514838802054417", "fe10e8d1b5fa5e23", "0251555cb1089f74"),
    (2, 6, 1, 260): ("2.126282821056321", "1c86f606ad655457", "a3e6800f5cca3db2"),
    (2, 6, 4, 260): ("2.353790945480625", "abb735783ae14007", "35ba7f672a6e7214"),
    (2, 6, 16, 260): ("2.5730349291071475", "27c6ba93e9877127", "3d1da1c8bbef97b9"),
    (2, 8, 1, 280): ("2.4931248072336385", "2f83fcad0271be6a", "254ea78c980be454"),
    (2, 8, 4, 280): ("2.6007518287800258", "d0f190bdc4948f60", "f57577fe14bb70a7"),
    (2, 8, 16, 280): ("2.6007518287800258", "3409b52ee7de58d1", "623e7d8d13c5cdc9"),
    (3, 4, 1, 340): ("2.3217079689886115", "7b4fd6b204800bcc", "15e8a613295c9fe0"),
    (3, 4, 4, 340): ("2.485270223169832", "7f501602f1271daf", "3e57cd1096430a6a"),
    (3, 4, 16, 340): ("2.5101438243873986", "32b25f2355988c07", "7f86ed99bd2e025d"),
    (3, 6, 1, 360): ("2.426440402616973", "22502b7ac913ae0b", "9fee6177837325fc"),
    (3, 6, 4, 360): ("2.5230047058117866", "8accf8e18f250db6", "e6d715463298424d"),
    (3, 6, 16, 360): ("2.5230047058117866", "013700d0c7cd59cb", "57d119479fec3b1b"),
    (3, 8, 1, 380): ("2.4269745348376315", "f62a3c6fbe0fcf65", "90fb9518731c84fa"),
    (3, 8, 4, 380): ("2.5558267428502757", "50d60afcfe54aaa0", "6726604112f1000d"),
    (3, 8, 16, 380): ("2.592796838574213", "85debfb4b12ab14e", "fd1b9eb01cd57745"),
    (2, 16, 64, 0): ("2.6496686308461896", "689664d4d0da6ca1", "a639b5e3184921ca"),
    (2, 3, 1000, 0): ("2.622894695402296", "9982f95b39870ed7", "32fb344d464a2c54"),
    (2, 16, 1024, 0): ("2.695257540796921", "3bfceec302cc2610", "0090f9b3edfb0b9b"),
    (3, 8, 64, 0): ("2.597501619808669", "3fce66cd73e8b71e", "92d17009453c853f"),
}


def records():
    return json.loads((GOLDEN / "golden.json").read_text())


def small_arrays():
    return np.load(GOLDEN / "small_cases.npz")


def case_input_soa(rec, oracle):
    """Haloed SoA input of a golden case, rebuilt from seed/const."""
    d, p, t = rec["d"], rec["p"], rec["t"]
    n, M, _ = oracle.sizes(d, p, t)
    if rec["const"] is not None:
        q = np.asarray(rec["const"], dtype=np.float64)
        return np.ascontiguousarray(np.repeat(q, t * M))
    return oracle.init_field_soa(d, p, t, rec["seed"], rec["gamma"])
