"""Engine-backed experiment harness: runs a reference
experiment JSON (configs/paper_figures/fig*.json key names, config.hpp:171-300)
through the B200 engine — every encode batch and prefill chunk executed on the
device — and writes report.csv (+ one Chrome trace per cell) in the reference's
schema (metrics.hpp report_csv_row / trace_to_json_text).

    python scripts/b200_experiment.py tests/golden/fig7_latency.json --out out/fig7_b200 \
        [--clock lockstep|real] [--model tiny|qwen2.5-vl-7b] [--ep] [--policies rserve,..]

--clock lockstep: the cost model orders events (the report must equal the
reference's byte for byte, which is checked when --golden is given);
--clock real: completions are CUDA-event timestamps of the executed work, so
the report is the hardware's figure. --ep runs the config's stages and
encoder_workers as separate EP ranks (loopback transport, one GPU).
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--out", required=True)
    ap.add_argument("--clock", default="lockstep", choices=["lockstep", "real"])
    ap.add_argument("--model", default="tiny")
    ap.add_argument("--ep", action="store_true")
    ap.add_argument("--policies", default=None)
    ap.add_argument("--rates", default=None)
    ap.add_argument("--seeds", default=None)
    ap.add_argument("--golden", default=None, help="report.csv to compare with (lockstep)")
    ap.add_argument("--traces", action="store_true", help="write one Chrome trace per cell")
    a = ap.parse_args()
    from paper_2509_24381_b200 import api
    cfg = json.load(open(a.config))
    wl, sim, policies, rates, seeds, slo = api.experiment_from_json(cfg)
    if a.policies:
        policies = a.policies.split(",")
    if a.rates:
        rates = [float(r) for r in a.rates.split(",")]
    if a.seeds:
        seeds = [int(s) for s in a.seeds.split(",")]
    m = api.model_preset(a.model)
    sim.hidden_size = m.llm_dim
    kw = dict(max_prompt_tokens=1 << 15, slot_tokens=1 << 19, kv_tokens=1 << 19, max_chunk_tokens=max(8192, sim.token_budget),
              max_encode_tokens=4096)
    ep = workers = None
    if a.ep:
        ranks = sim.stages + sim.encoder_workers
        ctxs = [api.ep_context(m, r, sim.stages, sim.encoder_workers, **kw) for r in range(ranks)]
        ctx, workers = ctxs[0], ctxs[1:]
        ep = api.EpGroup(sim.stages, sim.encoder_workers, "loopback")
    else:
        ctx = api.Pipeline(m, **kw)
    os.makedirs(a.out, exist_ok=True)
    rows = ["policy,rate,seed,mean_ttft_ms,p50,p90,p99,throughput_tok_s,slo_attainment"]
    launches, t0 = 0, time.time()
    for p in policies:
        for r in rates:
            for s in seeds:
                sim.policy = p
                wl.arrival_rate, wl.seed = r, s
                row, trace, st = api.engine_cell(ctx, wl, sim, slo, clock=a.clock, ep=ep, workers=workers)
                rows.append(row)
                launches += st["kernel_launches"]
                if a.traces:
                    with open(os.path.join(a.out, f"trace_{p}_{r:g}_{s}.json"), "w") as f:
                        f.write(trace)
                print(row, f"gpu_ms={st['gpu_ms']:.1f}", flush=True)
    with open(os.path.join(a.out, "report.csv"), "w") as f:
        f.write("\n".join(rows) + "\n")
    summary = dict(cells=len(rows) - 1, clock=a.clock, model=a.model, ep=a.ep, kernel_launches=launches,
                   wall_s=time.time() - t0)
    if a.golden:
        golden = open(a.golden).read().splitlines()
        summary["golden_identical"] = rows == golden[:len(rows)] if len(rows) < len(golden) else rows == golden
    print(json.dumps(summary))
    if a.golden and not summary["golden_identical"]:
        sys.exit(1)


if __name__ == "__main__":
    main()
