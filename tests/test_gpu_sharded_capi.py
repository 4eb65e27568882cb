"""The bond-sharded row absorb behind the C ABI (include/peps_b200.h:
pepsb_comm_init / pepsb_two_layer_apply_row_sharded /
pepsb_contract_two_layer_sharded; csrc/sharded.cpp) on one GPU: an NCCL
communicator of world size 1 (the collectives run, as identities, on the
library stream).  The multi-rank schedule itself is the one
paper_2006_15234_b200/sharded.py runs on world-size-2 gloo groups
(tests/test_sharded.py)."""
import numpy as np
import pytest

from conftest import rel
from oracle import peps_oracle as O
from paper_2006_15234_b200 import inputs as I

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm_ctx(A):
    ctx = A.Context(0)
    A.comm_init(ctx, A.comm_unique_id(), 0, 1)
    yield ctx
    A.comm_destroy(ctx)


@pytest.mark.parametrize("canon,key", [(True, "row_site"), (False, "row_split_site")])
def test_sharded_row_absorb_capi_matches_reference(A, golden, comm_ctx, canon, key):
    sites = I.random_peps(3, 5, 3, 71)
    top, phys = I.random_boundary(5, (3, 3), 9, 72)
    st = A.PepsState(3, 5, 2, sites, ctx=comm_ctx)
    tb = A.TwoLayerBoundary.from_sites(top, phys, ctx=comm_ctx)
    opt = A.ContractOption.two_layer_opt(9, 5, 2, -1)
    opt.canonicalize = canon
    out = A.two_layer_apply_row_sharded(tb, st, st, 1, opt, 0x20)
    assert out.phys == [(3, 3)] * 5
    for i, s in enumerate(out.sites):
        g = golden[f"{key}{i}"]
        assert s.shape == g.shape
        assert rel(s.numpy(), g) < 1e-8


def test_sharded_contract_two_layer_capi_matches_reference(A, refo, comm_ctx):
    sites = I.random_peps(5, 5, 2, 33, scale=0.5)
    st = A.PepsState(5, 5, 2, sites, ctx=comm_ctx)
    opt = A.ContractOption.two_layer_opt(6, 9, 2, -1)
    got = A.contract_two_layer_sharded(st, st, opt)
    want, _ = refo.contract_two_layer(sites, 5, 5, 6, 9, 2, -1)
    assert abs(got - want) <= 1e-8 * abs(want)
    # the unsharded device path agrees to rounding (different contraction order)
    assert abs(A.contract_two_layer(st, st, opt) - got) <= 1e-10 * abs(want)


def test_sharded_without_comm_is_a_validation_error(A):
    ctx = A.Context(0)
    sites = I.random_peps(3, 3, 2, 1)
    st = A.PepsState(3, 3, 2, sites, ctx=ctx)
    with pytest.raises(A.PepsError, match="ValidationError: no communicator"):
        A.contract_two_layer_sharded(st, st, A.ContractOption.two_layer_opt(4, 1, 1, -1))


def test_distributed_cached_environments_on_device(A, golden):
    """SURVEY §8(e) row 2 driver (sharded.distributed_local_expectations) with
    the device backend at world size 1: both sweeps, band environments and
    splices on the GPU; norm and the 16 <Z_i> + 4 <Z_iZ_j> against the
    reference's values (golden bands_*) to 1e-8."""
    from paper_2006_15234_b200 import sharded as SH
    sites = I.random_peps(4, 4, 2, 91, scale=1 / np.sqrt(8))
    terms = [tuple(int(x) for x in t) for t in golden["bands_terms"]]
    ops = SH.DeviceOps(SH.Comm())
    norm, vals = SH.distributed_local_expectations(ops, lambda c: SH.DeviceOps(c), [A.to_device(s) for s in sites],
                                                   4, 4, 4, 13, 2, -1, terms)
    assert abs(norm - golden["bands_norm"][0]) <= 1e-8 * abs(golden["bands_norm"][0])
    assert np.abs(vals - golden["bands_values"]).max() <= 1e-8


def test_sharded_deficient_grams_take_the_robust_path(A, refo, comm_ctx):
    """Bond-2 sites carrying a rank-1 product state: the probe Grams are
    deficient (the reference clamps and completes their columns,
    decomposition.cpp:86-117).  The stream-ordered sharded column detects the
    deficiency flags at its end and redoes the column on the robust path
    (counter faithful_redos); the norm still matches the reference."""
    rng = np.random.default_rng(5)
    sites = []
    for r in range(4):
        for c in range(4):
            shp = I.peps_site_shape(4, 4, r, c, 2)
            t = np.zeros(shp, dtype=complex)
            t[(slice(None),) + (0,) * 4] = rng.standard_normal(2)
            sites.append(t)
    st = A.PepsState(4, 4, 2, sites, ctx=comm_ctx)
    opt = A.ContractOption.two_layer_opt(8, 3, 2, -1)
    comm_ctx.reset_counters()
    got = A.contract_two_layer_sharded(st, st, opt)
    want, _ = refo.contract_two_layer(sites, 4, 4, 8, 3, 2, -1)
    assert abs(got - want) <= 1e-8 * abs(want)
    assert comm_ctx.counters()["faithful_redos"] > 0
