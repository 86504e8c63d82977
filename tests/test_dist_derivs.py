"""The closed-form feature derivatives of the device contact producer
(csrc/dist_derivs.cuh, host build) against the oracle's second-order duals
(the reference's distance.hpp arithmetic, pinned to oracle/_ref in
test_oracle_contact.py): on random and near-degenerate stencils, for the
region the classifier picks, the squared distance is bitwise the duals'
value and the gradient / Hessian agree to 1e-10 of their norms."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

import oracle_py as O

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def lib(tmp_path_factory):
    so = str(tmp_path_factory.mktemp("dd") / "libdd.so")
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-shared", "-fPIC", "-o", so,
                           os.path.join(HERE, "cpp", "dist_derivs_check.cpp")])
    L = C.CDLL(so)
    L.feat_derivs12.argtypes = [C.c_int, C.c_int] + [np.ctypeslib.ndpointer(np.float64, flags="C")] * 4
    return L


def closed_form(L, kind, region, x):
    v, g, H = np.zeros(1), np.zeros(12), np.zeros(144)
    L.feat_derivs12(kind, region, np.ascontiguousarray(x), v, g, H)
    return v[0], g, H.reshape(12, 12).T


def stencils(rng, n):
    for t in range(n):
        x = rng.normal(0, 1, 12)
        if t % 4 == 1:  # near-parallel edges / point near the triangle plane
            x[9:12] = x[6:9] + (x[3:6] - x[0:3]) + rng.normal(0, 1e-3, 3)
        if t % 4 == 2:
            x[0:3] = (x[3:6] + x[6:9] + x[9:12]) / 3 + rng.normal(0, 1e-4, 3)
        yield x


@pytest.mark.parametrize("kind", [0, 1])
def test_closed_form_equals_duals(lib, kind):
    rng = np.random.default_rng(10 + kind)
    regions = 7 if kind == 0 else 9
    seen = set()
    for x in stencils(rng, 400):
        d2, g, H = (O.pt_dist2_derivs if kind == 0 else O.ee_dist2_derivs)(x)
        matches = [r for r in range(regions) if closed_form(lib, kind, r, x)[0] == d2]
        assert matches, "no region reproduces the duals' value bitwise"
        v, gc, Hc = closed_form(lib, kind, matches[0], x)
        seen.add(matches[0])
        assert np.linalg.norm(gc - g) <= 1e-10 * np.linalg.norm(g) + 1e-300
        assert np.linalg.norm(Hc - H) <= 1e-10 * np.linalg.norm(H) + 1e-300
    assert len(seen) >= 3
