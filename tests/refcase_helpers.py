"""Model / feature builders for the reference-mirroring tests (the
reference's tests/helpers.py:135-195 shapes, restated for this package)."""
import numpy as np

from paper_2411_10143_b200 import FEATURE_NAMES
from paper_2411_10143_b200.inference import model_from_dict


def leaf(score):
    return {"score": float(score)}


def split(feature, threshold, left, right):
    idx = FEATURE_NAMES.index(feature) if isinstance(feature, str) else feature
    return {"feature_index": idx, "threshold": float(threshold), "left": left, "right": right}


def model_dict(classes, trees):
    return {"schema_version": 1, "feature_names": list(FEATURE_NAMES), "classes": classes,
            "trees": trees}


def stub_model(classes, forced):
    return model_from_dict(model_dict(classes, [[leaf(1.0 if c == forced else 0.0)] for c in classes]),
                           source="<stub>")


RANGES = {"nrows": (1, 300), "ncols": (1, 300), "nnz": (0, 27000), "density": (0, 1),
          "mean": (0, 90), "sd": (0, 40), "cov": (0, 5), "max": (0, 300), "min": (0, 300),
          "maxavg": (0, 300), "distavg": (0, 300), "clusteravg": (0, 300), "fill": (0, 50),
          "ndiag": (0, 600), "diagfill": (0, 50)}


def random_model(rng, classes, n_trees=8, depth=4):
    def node(level):
        if level == 0 or rng.random() < 0.3:
            return leaf(rng.normal())
        fi = int(rng.integers(0, len(FEATURE_NAMES)))
        lo, hi = RANGES[FEATURE_NAMES[fi]]
        return {"feature_index": fi, "threshold": float(rng.uniform(lo, hi)),
                "left": node(level - 1), "right": node(level - 1)}
    return model_from_dict(model_dict(classes, [[node(depth) for _ in range(n_trees)] for _ in classes]),
                           source="<random>")


def random_feature_array(rng):
    nrows, ncols = int(rng.integers(1, 300)), int(rng.integers(1, 300))
    nnz = int(rng.integers(0, nrows * ncols + 1))
    mean = nnz / nrows
    mx = float(rng.integers(0, ncols + 1))
    sd = float(rng.uniform(0, mx + 1))
    ndiag = float(rng.integers(0, nrows + ncols))
    return np.array([nrows, ncols, nnz, nnz / (nrows * ncols), mean, sd, sd / mean if mean else 0.0,
                     mx, float(rng.integers(0, mx + 1)), mx - mean, float(rng.uniform(0, ncols)),
                     float(rng.uniform(0, ncols)), nrows * mx / nnz if nnz else 0.0, ndiag,
                     nrows * ndiag / nnz if nnz else 0.0])
