"""Helpers to materialise the reference KATs (tests/golden/kats.json) and golden fixtures."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def kats():
    with open(os.path.join(GOLDEN, "kats.json")) as f:
        return json.load(f)


def trace(case):
    L, k = case["L"], case["k"]
    return np.asarray(case["choices"], np.int32).reshape(-1, L, k)


def dense_w(spec, m):
    W = np.zeros((m, m))
    if spec == "zero":
        return W
    for (j, k, v) in next(iter(spec.values())):
        W[j, k] = v
    return W


def e_from_nonzero(case):
    L, ne = case["L"], case["ne"]
    E = np.zeros((L - 1, ne, ne), np.uint64)
    for (l, j, k, v) in case["E_nonzero"]:
        E[l, j, k] = v
    return E


def expected_e(case):
    return e_from_nonzero(case)


def expected_w(case):
    ne = case["ne"]
    W = np.zeros((ne, ne), np.uint64)
    for (j, k, v) in case["W_nonzero"]:
        W[j, k] = v
    return W


def golden_cases():
    path = os.path.join(GOLDEN, "ref_cases.npz")
    z = np.load(path, allow_pickle=False)
    n = int(z["n_cases"])
    out = []
    for i in range(n):
        p = f"c{i}_"
        case = {key[len(p):]: z[key] for key in z.files if key.startswith(p)}
        out.append(case)
    return out
