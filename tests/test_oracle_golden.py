"""Generator + oracle against the SplitMix64 golden table of SURVEY.md §8(c).

Those values were computed during the survey by an independent scratch solver
(numpy SplitMix64 + a separate C kernel with the c1-c12 rules and c8
arithmetic), not by this repo's oracle — so agreement pins both the generator
(bit for bit) and the oracle's whole pivot path on the benchmark distribution.
Trace hash = SHA-256 of little-endian int32 (k, r) pairs, first 16 hex digits.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import lpgen
import oracle

GOLDEN_DIR = os.path.join(os.path.dirname(__file__), "golden")

# (m, n, seed): pivots, objective hex, first five (k, r), last (k, r), trace sha256[:16], nnz(x)
SURVEY_TABLE = {
    (64, 64, 1): (24, "0x1.c9320127cef55p+6", [(4, 45), (36, 63), (42, 11), (60, 41), (27, 7)],
                  (108, 61), "c0e8b78b69267088", 12),
    (64, 64, 2): (12, "0x1.a9e2d36d95463p+6", [(38, 23), (3, 38), (0, 20), (1, 15), (25, 8)],
                  (76, 45), "68762a76d845c33b", 9),
    (64, 64, 3): (39, "0x1.caf5ee56221e3p+6", [(57, 13), (18, 37), (20, 39), (5, 26), (45, 12)],
                  (12, 13), "947915a3d5ce01fe", 10),
    (1000, 1000, 1): (886, "0x1.c232e1a24b861p+10",
                      [(867, 747), (981, 905), (651, 935), (35, 50), (196, 119)],
                      (1448, 269), "4fe5601f55e0cfe0", 68),
    (4000, 4000, 1): (8487, "0x1.c74347d72074bp+12",
                      [(3508, 3007), (3194, 1433), (608, 641), (254, 1260), (3622, 2276)],
                      (609, 2476), "7467839cf994196f", 152),
    (8000, 8000, 1): (25395, "0x1.c8dbdb0fa38d5p+13",
                      [(3448, 3048), (6947, 5660), (5284, 5967), (2245, 4755), (6032, 7041)],
                      (10340, 5931), "71403ebd3a86721a", 242),
}


def trace_hash(k, r):
    return hashlib.sha256(np.stack([k, r], 1).astype("<i4").tobytes()).hexdigest()[:16]


def test_splitmix64_raw_outputs():
    # raw SplitMix64 outputs for seed 1
    z = lpgen.splitmix64(1, 0, 3)
    assert [int(v) for v in z] == [0x910a2dec89025cc1, 0xbeeb8da1658eec67, 0xf893a2eefb32555e]


def test_generator_first_values():
    A, b, c = lpgen.dense_lp(64, 64, 1)
    assert float(A[0, 0]).hex() == "0x1.8656e75434454p+2"
    assert float(A[0, 1]).hex() == "0x1.ed91feab24819p+2"
    assert float(b[0]).hex() == "0x1.d3678a882fc32p+6"
    assert float(c[0]).hex() == "0x1.1c18f863c4850p+3"
    A, b, c = lpgen.dense_lp(1000, 1000, 1)
    assert float(b[0]).hex() == "0x1.1242f5d138a7fp+10"
    assert float(c[0]).hex() == "0x1.0961a272f4392p+3"


def test_generator_counter_based_blocks():
    A, _, _ = lpgen.dense_lp(50, 40, 9)
    assert np.array_equal(lpgen.dense_A_rows(50, 40, 9, 17, 33), A[17:33])
    assert A.min() >= 1.0 and A.max() < 10.0


@pytest.mark.parametrize("key", [(64, 64, 1), (64, 64, 2), (64, 64, 3), (1000, 1000, 1)])
def test_oracle_matches_survey_golden(key):
    pivots, objhex, first5, last, h, nnz = SURVEY_TABLE[key]
    A, b, c = lpgen.dense_lp(*key)
    res = oracle.solve(A, b, c)
    assert res.status == oracle.OPTIMAL
    assert res.pivots == pivots
    assert float(res.objective).hex() == objhex
    assert res.trace()[:5] == first5 and res.trace()[-1] == last
    assert trace_hash(res.trace_k, res.trace_r) == h
    assert int((res.x != 0).sum()) == nnz
    cert = oracle.certificate(A, b, c, res.x, res.y)
    assert not cert.violations, cert.violations


@pytest.mark.parametrize("key", [(64, 64, 1), (1000, 1000, 1), (4000, 4000, 1), (8000, 8000, 1)])
def test_stored_golden_files_match_survey(key):
    # tests/golden/*.npz are written by scripts/make_golden.py (oracle only); the
    # large ones take the oracle minutes to hours, so the GPU parity tests read them.
    path = os.path.join(GOLDEN_DIR, "dense_%dx%d_s%d.npz" % key)
    if not os.path.exists(path):
        pytest.skip("golden file not generated yet: " + path)
    g = np.load(path)
    pivots, objhex, first5, last, h, nnz = SURVEY_TABLE[key]
    assert int(g["pivots"]) == pivots
    assert float(g["objective"]).hex() == objhex
    assert trace_hash(g["trace_k"], g["trace_r"]) == h
    assert int(g["x_idx"].size) == nnz
    meta = json.load(open(path[:-4] + ".json"))
    assert meta["trace_sha256_16"] == h
