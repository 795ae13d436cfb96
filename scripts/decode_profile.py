"""Per-kernel-class device time of greedy decode on the cfg2 request (7B,
8.6k context, batch 1): profiler events around every launch.

  python scripts/decode_profile.py [steps]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2509_24381_b200 import _native as N  # noqa: E402
from paper_2509_24381_b200 import api  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 16
mcfg = api.model_preset("qwen2.5-vl-7b")
m = {k: getattr(mcfg, k) for k, _ in N.rs_model_config._fields_}
pipe = api.Pipeline(mcfg, max_prompt_tokens=bench.MAX_PROMPT, slot_tokens=1 << 16, kv_tokens=1 << 16,
                    max_chunk_tokens=2048, max_encode_tokens=1024)
wl = f"0,0,-,{bench.LAYOUT}\n"
sc = bench.sim_cfg(argparse.Namespace(policy="rserve", budget=2048), m)
pipe.run(wl, sc, clock="real", payload_seed=1234, keep_kv=True)
pipe.decode([0], 4)
_, _, ms_plain = pipe.decode([0], steps)
N.check(N.lib.rs_profile_enable(1))
_, _, ms_prof = pipe.decode([0], steps)
N.check(N.lib.rs_profile_enable(0))
prof = N.profile_drain()
pipe.decode_release(0)
pipe.close()
rows = sorted(((k, v["launches"] / steps, v["ms"] / steps * 1e3) for k, v in prof.items()), key=lambda r: -r[2])
print(json.dumps({"tpot_ms": ms_plain / steps, "tpot_ms_profiled": ms_prof / steps,
                  "per_step_us": [(k, round(n, 1), round(us, 1)) for k, n, us in rows]}, indent=1))
