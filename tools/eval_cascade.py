"""Timing regret of cascade model sets on a labelled B200 dataset (build-time
tool): for every matrix of DATASET (its FORMAT.csv feature rows and cached
timing tables), the SpMV time of the configuration each model set predicts,
relative to the fastest configuration, geometric mean per family.

    python tools/eval_cascade.py DATASET MODELS_DIR [MODELS_DIR ...]
"""
import json
import math
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from paper_2411_10143_b200.features import FEATURE_NAMES, FeatureVector  # noqa: E402
from paper_2411_10143_b200.inference import CascadeModelSet, cascade_predict  # noqa: E402

ds = Path(sys.argv[1])
rows = [ln for ln in (ds / "FORMAT.csv").read_text().splitlines()[2:]]
cache = {json.loads(f.read_text())["matrix_id"]: json.loads(f.read_text())["times"]
         for f in (ds / "cache").glob("*.json")}
ids = list(cache)
ids = sorted(ids, key=lambda i: int(i.rsplit("_", 1)[-1])) if all(
    i.rsplit("_", 1)[-1].isdigit() for i in ids) else sorted(ids)
assert len(ids) == len(rows)
sets = {"default CSR/LibA/32": None}
for d in sys.argv[2:]:
    sets[d] = CascadeModelSet.load_dir(d)
res = {k: defaultdict(list) for k in sets}
for mid, ln in zip(ids, rows):
    vals = [float(v) for v in ln.split(",")[:-1]]
    fv = FeatureVector(**dict(zip(FEATURE_NAMES, vals)))
    times = {k: v for k, v in cache[mid].items() if v}
    best = min(times.values())
    fam = mid.split("_")[0]
    for name, ms in sets.items():
        tok = "CSR/LibA/32" if ms is None else cascade_predict(ms, fv).token()
        t = times.get(tok, max(times.values()))
        res[name][fam].append(t / best)
        res[name]["ALL"].append(t / best)
fams = sorted({f for r in res.values() for f in r})
print(f"{'model set':40s} " + " ".join(f"{f:>10s}" for f in fams))
for name, r in res.items():
    print(f"{name[-40:]:40s} " + " ".join(f"{math.exp(np.mean(np.log(r[f]))):10.3f}" for f in fams))
