"""Loader for tests/golden/golden.npz (made by tests/golden/make_golden.py
from the unmodified reference)."""

import os
from functools import lru_cache

import numpy as np

from oracle.oracle import Csr

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.npz")


@lru_cache(maxsize=1)
def golden():
    with np.load(PATH) as z:
        return {k: z[k] for k in z.files}


def csr(key: str) -> Csr:
    G = golden()
    return Csr.of(int(G[f"{key}/n"]), G[f"{key}/node_pointer"], G[f"{key}/edge_list"],
                  G.get(f"{key}/values"))


def transform(key: str, geom="16x8") -> dict:
    G = golden()
    p = f"{key}/t{geom}/"
    return {k[len(p):]: v for k, v in G.items() if k.startswith(p)}


def random_keys():
    return sorted({k.split("/")[0] for k in golden() if k.startswith("rand") and "_" not in k.split("/")[0]})
