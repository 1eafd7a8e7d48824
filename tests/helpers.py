"""Shared test helpers: golden-fixture loaders and the parity metrics of the contract
(SURVEY.md 8c): rel 1e-4 per sweep, Frobenius and max-abs / max|ref|."""

from __future__ import annotations

import json

import numpy as np


def rel_errors(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    fro = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300)
    mx = np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-300)
    return float(fro), float(mx)


def assert_rel(got, ref, tol=1e-4, what=""):
    fro, mx = rel_errors(got, ref)
    assert fro <= tol and mx <= tol, f"{what}: rel fro {fro:.3e} max {mx:.3e} > {tol:g}"
    return fro, mx


def manifest(z):
    return json.loads(bytes(z["manifest"]).decode())


def model_arrays(z, prefix, N):
    return ([np.array(z[f"{prefix}A{n}"]) for n in range(N)],
            [np.array(z[f"{prefix}B{n}"]) for n in range(N)])
