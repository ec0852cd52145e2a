"""Retrain the cascade on B200 timings — BUILD-TIME
TOOL, run in the build container only (it imports the reference's offline
trainer from /root/reference/pkg/trainer; nothing at run time does).

    python -m paper_2411_10143_b200 dataset --generated 210 --seed 1 --out DS   # on the B200
    python tools/retrain_b200.py DS paper_2411_10143_b200/models/b200

Per stage dataset (reference trainer/train.py:87-121 via `train_one`):
rows whose best and second-best stage candidates (from the cached per-matrix
B200 timing tables) are within --tie of each other are dropped before
training, since on the GPU those labels are timing noise; a stage whose
dataset has a single class gets a constant model (the trainer requires two
classes).  Writes the five model files in the reference schema plus
provenance.json (dataset fingerprint, row counts, held-out accuracy).
"""
from __future__ import annotations

import argparse
import json
import shutil
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def dataset_order(ids):
    """Row order of build_dataset's CSVs: generation order for a generated
    corpus (ids end in _<index>), file-name order for a .mtx directory."""
    ids = list(ids)
    if ids and all(i.rsplit("_", 1)[-1].isdigit() for i in ids):
        return sorted(ids, key=lambda i: int(i.rsplit("_", 1)[-1]))
    return sorted(ids)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("dataset")
    ap.add_argument("out")
    ap.add_argument("--tie", type=float, default=0.03, help="relative gap below which a label is noise")
    ap.add_argument("--trees", type=int, default=60)
    ap.add_argument("--depth", type=int, default=3)
    args = ap.parse_args()
    tmp = Path(tempfile.mkdtemp())
    shutil.copytree("/root/reference/pkg/trainer/src/spmv_trainer", tmp / "spmv_trainer")
    sys.path.insert(0, str(tmp))
    sys.path.insert(0, "/root/reference/pkg/src")
    import pandas as pd
    from spmv_trainer.schema import FEATURE_NAMES, dump_model
    from spmv_trainer.train import TrainConfig, read_dataset, train_one

    from paper_2411_10143_b200.harness import DATASET_FILES, SpmvConfig, label_from_times  # noqa: F401

    ds = Path(args.dataset)
    out = Path(args.out)
    out.mkdir(parents=True, exist_ok=True)
    # per-matrix stage margins from the timing cache
    cache = {}
    for f in sorted((ds / "cache").glob("*.json")):
        d = json.loads(f.read_text())
        cache[d["matrix_id"]] = d["times"]

    def margins(times):
        def t(tok):
            return times.get(tok)
        lane = [t(f"CSR/LibA/{w}") for w in (2, 4, 8, 16, 32)]
        lane = min(v for v in lane if v) if any(lane) else None
        stages = {
            "FORMAT": [lane, t("COO/LibA"), t("ELL/LibA"), t("DIA/LibA"), t("HYB/LibA")],
            "COO-LIB": [t("COO/LibA"), t("COO/LibB")],
            "CSR-LIB": [lane, t("CSR/LibB"), t("CSR/LibC")],
            "ELL-LIB": [t("ELL/LibA"), t("ELL/LibC")],
            "CSR-TPV": [t(f"CSR/LibA/{w}") for w in (2, 4, 8, 16, 32)],
        }
        res = {}
        for k, vals in stages.items():
            v = sorted(x for x in vals if x)
            res[k] = (v[1] - v[0]) / v[0] if len(v) > 1 else float("inf")
        return res

    # the CSVs keep matrix order; recover ids from the cache order used by build_dataset
    prov = {"dataset": str(ds), "tie": args.tie, "trees": args.trees, "depth": args.depth, "models": {}}
    fp = (ds / "FORMAT.csv").read_text().splitlines()[0]
    prov["fingerprint"] = fp
    ids_in_order = dataset_order(cache)
    routes = {name: [] for name in DATASET_FILES}
    from paper_2411_10143_b200.harness import route_labels
    for mid in ids_in_order:
        try:
            lab = label_from_times(cache[mid])
        except Exception:
            continue
        for name in route_labels(lab):
            routes[name].append(mid)
    cfg = TrainConfig(n_trees=args.trees, max_depth=args.depth)
    for name, fname in DATASET_FILES.items():
        frame = read_dataset(ds / fname)
        mids = routes[name]
        assert len(mids) == len(frame), (name, len(mids), len(frame))
        keep = [margins(cache[m])[name] >= args.tie for m in mids]
        frame = frame[pd.Series(keep, index=frame.index)].reset_index(drop=True)
        classes = sorted(frame["label"].unique()) if len(frame) else []
        if len(classes) >= 2:
            doc, met, _ = train_one(frame, cfg, name)
            info = met.to_dict()
        else:
            only = classes[0] if classes else ("LibA" if name != "CSR-TPV" else "32")
            doc = {"classes": [only], "feature_names": list(FEATURE_NAMES), "schema_version": 1,
                   "trees": [[{"score": 0.0}]]}
            info = {"constant": only}
        info["rows_after_tie_filter"] = int(len(frame))
        info["rows_total"] = len(mids)
        dump_model(doc, out / f"{name}.json")
        prov["models"][name] = info
        print(name, info)
    (out / "provenance.json").write_text(json.dumps(prov, indent=1) + "\n")


if __name__ == "__main__":
    main()
