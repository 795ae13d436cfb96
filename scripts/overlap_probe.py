"""cfg2 step with the encoder on its own high-priority stream (real clock, the
bench's mode) vs the encoder serialised onto the prefill stream, device ms.

  python scripts/overlap_probe.py [reps]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2509_24381_b200 import _native as N  # noqa: E402
from paper_2509_24381_b200 import api  # noqa: E402
import argparse  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
mcfg = api.model_preset("qwen2.5-vl-7b")
m = {k: getattr(mcfg, k) for k, _ in N.rs_model_config._fields_}
pipe = api.Pipeline(mcfg, max_prompt_tokens=bench.MAX_PROMPT, slot_tokens=1 << 19, kv_tokens=1 << 19,
                    max_chunk_tokens=2048, max_encode_tokens=1024)
wl = f"0,0,-,{bench.LAYOUT}\n"
ns = argparse.Namespace(policy="rserve", budget=2048)
sc = bench.sim_cfg(ns, m)
sc_ser = bench.sim_cfg(ns, m, beta_enc=0.0001)
out = {}
for name, kw in (("concurrent_real", dict(clock="real")), ("serialized_lockstep", dict(clock="lockstep", serialize=True)),
                 ("concurrent_lockstep", dict(clock="lockstep"))):
    s = sc if name == "concurrent_real" else sc_ser
    for _ in range(2):
        pipe.run(wl, s, payload_seed=1234, **kw)
    ms = []
    for _ in range(reps):
        _, _, st = pipe.run(wl, s, payload_seed=1234, **kw)
        ms.append(st["gpu_ms"])
    ms.sort()
    out[name] = {"gpu_ms_p50": ms[len(ms) // 2], "all": [round(x, 2) for x in ms]}
print(json.dumps(out))
pipe.close()
