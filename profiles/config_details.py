"""bench.py's config 1/2/3 detail legs on their own (no config-5 run): the
async / sequential / default solves and the per-kernel roofline of config 2.
    python profiles/config_details.py [config2 config1 config3]"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402

which = sys.argv[1:] or ["config2"]
import paper_2411_10143_b200 as P  # noqa: E402
from paper_2411_10143_b200 import _lib, device  # noqa: E402
models = P.CascadeModelSet.load_dir(ROOT / "tests" / "golden" / "models")
args = argparse.Namespace(steps=10, warmup=3)
fns = {"config2": bench.config2_detail, "config1": bench.config1_detail, "config3": bench.config3_detail}
for name in which:
    print(json.dumps({name: fns[name](args, P, device, _lib, models)}), flush=True)
