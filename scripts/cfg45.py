"""north_star configs 4 and 5 on ONE B200 (bench.py run_cfg4 / run_cfg5; the
bench's N = 1 line carries the same blocks). cfg4 = the C sweep 128-2048
(experiment.hpp:296-330) over the cfg3 request stream; cfg5 = the video-frame
workload (ConsecutiveMm, 64 x M256 + T128) on the 72B-shaped LLM. Both
co-located on one GPU: their 4E+4P placement needs eight.

  python scripts/cfg45.py [cfg4] [cfg5] [--steps K] > cfg45.json
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", nargs="*", default=["cfg4", "cfg5"])
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    out = {}
    if "cfg4" in args.which:
        out["cfg4"] = bench.run_cfg4(args.steps)
    if "cfg5" in args.which:
        out["cfg5"] = bench.run_cfg5(args.steps)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
