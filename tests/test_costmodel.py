"""CPU: the algorithmic flop model used for bench.py's TFLOP/s reproduces the
reference's own instr::flops counter exactly (instrument.hpp:19-65)."""
import pytest

from paper_2006_15234_b200 import costmodel as CM
from paper_2006_15234_b200 import inputs as I


@pytest.mark.parametrize("L,r,m,q,os_", [(4, 2, 4, 1, 4), (5, 3, 9, 2, -1), (6, 4, 16, 2, 8)])
def test_row_absorb_flops_match_reference_counter(refo, L, r, m, q, os_):
    sites = I.random_peps(3, L, r, 7)
    top, phys = I.random_boundary(L, (r, r), m, 8)
    _, _, info = refo.two_layer_apply_row(top, phys, sites, 3, L, 1, m, 5, q, os_)
    assert CM.two_layer_row_flops(L, r, m, q, os_) == int(info["flops"])


def test_rsvd_flops_match_reference_counter(refo):
    v = I.gaussian((8, 3, 3, 8, 3, 3), 1)
    s = I.gaussian((3, 3, 8, 8), 2)
    b = I.gaussian((2, 3, 3, 3, 3), 3)
    ts, labs = [v, s, b.conj(), b], ["apqsmn", "uvst", "dumbe", "dvncf"]
    out = refo.einsumsvd(ts, labs, "apq", "bctef", 8, 1e-14, "implicit_rsvd", "left", 2, 8, 5)
    assert CM.rsvd_flops([t.shape for t in ts], labs, "apq", "bctef", 8, 2, 8) == int(out["flops"])


def test_config2_count_matches_baseline_md():
    # one config-2 row absorb counts 6.876e11 reference flops
    assert CM.two_layer_row_flops(8, 8, 64, 2, 8) == 687608257024
