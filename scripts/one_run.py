"""One lock-step engine run of the cfg2 request on the 7B-shaped model (for
ncu captures of the tracker / KV kernels at bench shapes)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_24381_b200 import api  # noqa: E402

LAYOUT = "T128|" + "|".join(["M1024|T32"] * 8)
m = api.model_preset("qwen2.5-vl-7b")
pipe = api.Pipeline(m, max_prompt_tokens=16384, slot_tokens=1 << 15, kv_tokens=1 << 15,
                    max_chunk_tokens=2048, max_encode_tokens=1024)
sc = api.SimConfig(policy="rserve", stages=1, token_budget=2048, embedding_batch_tokens=1024,
                   encoder_workers=1, hidden_size=m.llm_dim,
                   cost=api.CostModel(beta_enc_ms_per_token=0.0001, delta_stage_ms_per_token=0.01))
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    pipe.run(f"0,0,-,{LAYOUT}\n", sc, clock="lockstep", payload_seed=1234)
pipe.close()
print("ok")
