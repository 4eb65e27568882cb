"""The JSON front ends over the device:
run_expect_json (drivers.cpp:509-550) reading the reference's own PEPS
container, run_vqe_json / run_vqe (drivers.cpp:134-191, 384-425) with the
Nelder-Mead and COBYLA-lite loops of optimize.cpp, run_ite_json
(drivers.cpp:335-382); every result document against the compiled
reference's on the same config."""
import json

import numpy as np
import pytest

from paper_2006_15234_b200 import drivers as D
from paper_2006_15234_b200 import inputs as I

pytestmark = pytest.mark.gpu


def _close(a, b, tol=1e-8):
    return abs(a - b) <= tol * max(1.0, abs(b))


@pytest.mark.parametrize("ham", [
    {"type": "j1j2", "j1": 1.0, "j2": 0.3, "h": [0.4, 0.0, 0.2]},
    {"type": "text", "terms": "-1.0 Z@(0,0) Z@(0,1)\n-1.0 Z@(1,0) Z@(2,0)\n-3.0 X@(1,1)\n0.5 Y@(2,2) Y@(2,1)"},
])
@pytest.mark.parametrize("family,shared", [("two-layer-ibmps", False), ("two-layer-ibmps", True), ("bmps", True)])
def test_run_expect_json_matches_reference(A, refo, tmp_path, ham, family, shared):
    sites = I.random_peps(3, 3, 2, 77, scale=0.5)
    path = str(tmp_path / "state.peps")
    refo.save_peps(sites, 3, 3, path)  # the reference writes the container; the device reads it
    cfg = json.dumps({"schema": 1, "state": path, "hamiltonian": ham, "family": family, "m": 8, "rsvd_iters": 2,
                      "seed": 11, "shared_environments": shared})
    got = json.loads(D.run_expect_json(cfg))
    want = json.loads(refo.json_driver("expect", cfg))
    assert got["schema"] == want["schema"] == 1 and got["command"] == want["command"] == "expect"
    assert got["config"] == want["config"] and got["versions"] == want["versions"]
    g, w = got["results"], want["results"]
    for k in ("value", "value_per_site", "raw_sum_re", "raw_sum_im", "norm_sq"):
        assert _close(g[k], w[k]), (k, g[k], w[k])
    assert g["full_sweeps"] == w["full_sweeps"] and g["band_contractions"] == w["band_contractions"]


def test_run_expect_json_observable_file(A, refo, tmp_path):
    sites = I.random_peps(2, 3, 2, 5, scale=0.7)
    path = str(tmp_path / "s.peps")
    refo.save_peps(sites, 2, 3, path)
    obs = tmp_path / "obs.txt"
    obs.write_text("# two terms\n0.7 X@(0,1)\n-1.0 Z@(0,0) Z@(1,0)\n")
    cfg = json.dumps({"schema": 1, "state": path, "observable_file": str(obs), "m": 6})
    g = json.loads(D.run_expect_json(cfg))["results"]
    w = json.loads(refo.json_driver("expect", cfg))["results"]
    assert _close(g["value"], w["value"]) and _close(g["norm_sq"], w["norm_sq"])


@pytest.mark.parametrize("opt,init", [("nelder-mead", "random"), ("cobyla", "neel")])
def test_run_vqe_json_matches_reference(A, refo, opt, init):
    """Same seeded theta0, same objective values (1e-8) -> the optimizer takes the
    same path: evaluation count, trace and best theta agree."""
    cfg = json.dumps({"schema": 1, "rows": 2, "cols": 2, "layers": 1, "init": init,
                      "optimizer": {"name": opt, "max_evaluations": 14, "initial_step": 0.4},
                      "evolution_rank": 2, "contraction_rank": 4, "seed": 3,
                      "hamiltonian": {"type": "j1j2", "j1": [0.0, 0.0, 1.0], "h": [0.8, 0.0, 0.0]}})
    g = json.loads(D.run_vqe_json(cfg))["results"]
    w = json.loads(refo.json_driver("vqe", cfg))["results"]
    assert g["evaluations"] == w["evaluations"] == 14
    np.testing.assert_allclose(g["trace"], w["trace"], rtol=1e-8, atol=1e-10)
    np.testing.assert_allclose(g["running_minimum"], w["running_minimum"], rtol=1e-8, atol=1e-10)
    np.testing.assert_allclose(g["best_theta"], w["best_theta"], rtol=1e-8, atol=1e-10)
    assert _close(g["best_energy"], w["best_energy"])


def test_run_ite_json_matches_reference(A, refo):
    cfg = json.dumps({"schema": 1, "rows": 3, "cols": 3, "tau": 0.05, "steps": 4, "evolution_rank": 2,
                      "contraction_rank": 8, "rsvd_iters": 2, "energy_every": 2, "initial": "neel", "seed": 1,
                      "hamiltonian": {"type": "j1j2", "j1": [0.0, 0.0, 1.0], "h": [2.0, 0.0, 0.0]}})
    g = json.loads(D.run_ite_json(cfg))["results"]
    w = json.loads(refo.json_driver("ite", cfg))["results"]
    assert [e["step"] for e in g["energies"]] == [e["step"] for e in w["energies"]] == [2, 4]
    for a, b in zip(g["energies"], w["energies"]):
        assert _close(a["energy"], b["energy"]), (a, b)
    assert g["final_max_bond"] == w["final_max_bond"]
