"""The full-size oracle goldens (tests/golden/oracle_C*.json, tools/make_oracle_golden.py) are current and
self-consistent (CPU, -m "not gpu").

  * each file's oracle_source_sha256 equals the hash of today's oracle/ + inputs/ sources, so a golden can never
    silently outlive a change of the oracle's arithmetic (regenerate with the tool when this fails);
  * the generator reproduces the C1 golden in-process (C1 is small enough to rerun here);
  * structural facts the goldens must satisfy: columns = sum of per-cycle columns = len(hist_est); the restarted
    configs end at or below tol and only there (O15/O16); every cycle but the last ends above tol;
  * C5: the top Ritz value lies within 1e-3 of the closed-form largest eigenvalue of the Kronecker-sum stencil
    (a fact independent of the oracle's code path), and the Ritz list is in the canonical order of reading O23.
"""
import importlib.util
import json
import os

import numpy as np
import pytest

import oracle as O
from inputs import get_config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def _tool():
    spec = importlib.util.spec_from_file_location("mog", os.path.join(ROOT, "tools", "make_oracle_golden.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _load(name):
    with open(os.path.join(GOLDEN, f"oracle_{name}.json")) as fh:
        return json.load(fh)


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5", "C5B"])
def test_golden_is_current(name):
    g = _load(name)
    assert g["oracle_source_sha256"] == _tool().source_hash(g["method"]), \
        f"oracle/ or inputs/ changed since oracle_{name}.json was written: rerun tools/make_oracle_golden.py {name}"


def test_c1_golden_reproduces():
    g = _load("C1")
    r = _tool().run_sgmres(get_config("C1"))
    assert (r["cycles"], r["columns"]) == (g["cycles"], g["columns"])
    np.testing.assert_allclose(r["hist_est"], g["hist_est"], rtol=1e-10)
    np.testing.assert_allclose(r["x_sample"], g["x_sample"], rtol=1e-10, atol=1e-14)
    assert abs(r["rel_res_true"] - g["rel_res_true"]) <= 1e-10 * g["rel_res_true"]


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_sgmres_golden_structure(name):
    cfg = get_config(name)
    g = _load(name)
    assert g["columns"] == sum(g["columns_per_cycle"]) == len(g["hist_est"])
    assert len(g["hist_true"]) == g["cycles"] == len(g["columns_per_cycle"])
    assert all(1 <= c <= cfg.d for c in g["columns_per_cycle"])
    assert g["rel_res_true"] == g["hist_true"][-1]
    if cfg.max_cycles > 1:
        assert g["rel_res_true"] <= cfg.tol
        assert all(h > cfg.tol for h in g["hist_true"][:-1])
    assert len(g["x_sample_rows"]) == len(g["x_sample"]) == min(64, cfg.n)


def test_srr_golden_structure():
    cfg = get_config("C5")
    g = _load("C5")
    th = np.asarray(g["theta_re"]) + 1j * np.asarray(g["theta_im"])
    assert len(th) >= cfg.nev
    lam_max = O.closed_form_eigs(2, cfg.m, cfg.beta).max()
    assert abs(th[0].real - lam_max) <= 1e-3 * lam_max
    assert np.array_equal(O.select_ritz(th, len(th)), np.arange(len(th)))     # canonical order (O23)
    assert np.all(np.asarray(g["res_true"]) > 0) and np.all(np.asarray(g["res_est"]) > 0)
