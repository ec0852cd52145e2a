"""Loaders for the golden fixtures written by tests/golden/make_golden.py."""
from __future__ import annotations

import json
from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(maxsize=None)
def index():
    return json.loads((GOLDEN / "index.json").read_text())


def case_names():
    return [c["name"] for c in index()["cases"]]


@lru_cache(maxsize=None)
def case(name):
    with np.load(GOLDEN / "cases" / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


@lru_cache(maxsize=None)
def cascade_doc():
    return json.loads((GOLDEN / "cascade.json").read_text())


@lru_cache(maxsize=None)
def solves():
    return json.loads((GOLDEN / "solves.json").read_text())


def model_docs():
    return {p.stem: json.loads(p.read_text()) for p in sorted((GOLDEN / "models").glob("*.json"))}


def spmv_keys(c):
    """(token, workers) pairs stored for a case."""
    out = []
    for k in c:
        if k.startswith("y|"):
            _, tok, w = k.split("|")
            out.append((tok, int(w)))
    return out
