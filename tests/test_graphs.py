"""The product-side restatement of the reference's generators
(graphs.reference_random_csr / reference_random_dense, used by bench.py for
BASELINE configs[0]/[1]) must reproduce the reference's own C1 inputs: the
golden hashes come from the compiled reference (tests/golden/make_golden.py)."""
import json
import pathlib
import sys

import pytest

sys.path.insert(0, str(pathlib.Path(__file__).parent / "golden"))
import cases  # noqa: E402

from paper_2412_11007_b200 import graphs as G  # noqa: E402

GOLD = json.loads((pathlib.Path(__file__).parent / "golden" / "golden.json").read_text())["cases"]


@pytest.mark.parametrize("name,kind", [("c1", "int"), ("c1_real", "real")])
def test_reference_generators_reproduce_c1(name, kind):
    rp, ci, v = G.reference_random_csr(4096, 4096, 16.0 / 4096, 1, kind)
    assert ci.size == 64899
    assert cases.sha(rp, ci, v) == GOLD[name]["csr"]
    for key, seed, shape in (("B", 2, (4096, 128)), ("A", 3, (4096, 32)), ("Bt", 4, (4096, 32))):
        assert cases.sha(G.reference_random_dense(*shape, seed, kind)) == GOLD[name][key]["sha"], key


def test_reference_generator_small_cases_match_oracle():
    import oracle as O
    for rows, cols, dens, seed in ((1, 1, 1.0, 3), (7, 13, 0.3, 11), (33, 5, 0.9, 12345), (64, 64, 0.01, 7)):
        m = O.generate_random_sparse(rows, cols, dens, seed)
        rp, ci, v = G.reference_random_csr(rows, cols, dens, seed)
        assert (rp == m.row_ptr).all() and (ci == m.col_idx).all() and (v == m.values).all()
