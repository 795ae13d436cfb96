"""Payload files restated for the oracle — TEST
INFRASTRUCTURE, an independent reading of the format the product parses in
paper_2509_24381_b200/csrc/payload.cu (host/payload.hpp):

    # rserve payload v1
    <req_id>,<segment_index>,M,grid=<gh>x<gw>[;seed=<u64>]
    <req_id>,<segment_index>,T,seed=<u64> | ids=<id> <id> ...

resolve() turns one request's lines into what the model consumes: per image
its merged-token grid and pixel seed, and the text token ids in prompt order
(defaults: the most square grid, the run's payload seed, hashed ids —
model_oracle.token_ids / item_grid, mirroring the reference-layout-only
workload files of workload.hpp:217-265)."""
from typing import Dict

import numpy as np

from . import model_oracle as mo


def parse(text: str) -> Dict[int, Dict]:
    out: Dict[int, Dict] = {}
    for line in text.splitlines():
        t = line.strip()
        if not t or t.startswith("#"):
            continue
        rid, seg, kind, spec = (x.strip() for x in t.split(",", 3))
        r = out.setdefault(int(rid), {"M": {}, "T": {}})
        if kind == "M":
            d = {}
            for kv in spec.split(";"):
                k, v = kv.split("=")
                if k == "grid":
                    gh, gw = v.split("x")
                    d["grid"] = (int(gh), int(gw))
                else:
                    d["seed"] = int(v)
            r["M"][int(seg)] = d
        else:
            k, v = spec.split("=", 1)
            r["T"][int(seg)] = {"ids": [int(x) for x in v.split()]} if k == "ids" else {"seed": int(v)}
    return out


def resolve(layout: str, req_id: int, spec: Dict, run_seed: int, vocab: int) -> Dict:
    segs = mo.parse_layout(layout)
    grids, seeds, ids = [], [], []
    pos = 0
    for s, (kind, n) in enumerate(segs):
        if kind == "M":
            d = spec.get("M", {}).get(s, {}) if spec else {}
            grids.append(d.get("grid", mo.item_grid(n)))
            seeds.append(d.get("seed", run_seed))
        else:
            d = spec.get("T", {}).get(s, {}) if spec else {}
            if "ids" in d:
                ids.extend(d["ids"])
            else:
                p = np.arange(pos, pos + n, dtype=np.int64)
                ids.extend(mo.token_ids(d.get("seed", run_seed), req_id, p, vocab).tolist())
        pos += n
    return {"item_grids": grids, "item_seeds": seeds, "text_ids": ids}
