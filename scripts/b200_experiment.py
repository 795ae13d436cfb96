"""Engine-backed experiment harness: runs a reference
experiment JSON (configs/paper_figures/fig*.json key names, config.hpp:171-300)
through the B200 engine — every encode batch and prefill chunk executed on the
device — and writes the reference's outputs in the reference's schema:

    run                report.csv (+ one Chrome trace per cell), run_experiment
                       (experiment.hpp:109-173; metrics.hpp report_csv_row)
    compare            per-rate comparison of two policies over matching
                       (rate, seed) cells, compare_policies (experiment.hpp:222-281)
    sweep-batch-size   mean TTFT / throughput per embedding batch size C,
                       policies[0] at rates[0] averaged over the seeds,
                       batch_size_sweep.csv, sweep_batch_size (experiment.hpp:296-330)

    python scripts/b200_experiment.py tests/golden/fig7_latency.json --out out/fig7_b200 \\
        [run|compare --baseline epd_baseline --target rserve|sweep-batch-size --values 128,256]
        [--clock lockstep|real] [--model tiny|qwen2.5-vl-7b] [--ep] [--policies rserve,..]

--clock lockstep: the cost model orders events (the outputs must equal the
reference's byte for byte, checked when --golden is given; tests/
test_experiment_gpu.py); --clock real: completions are CUDA-event timestamps
of the executed work, so the outputs are the hardware's figures. --ep runs
the config's stages and encoder_workers as separate EP ranks (loopback
transport, one GPU).
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

WHOLE_REQUEST = 0xFFFFFFFFFFFFFFFF


def fmt(v: float) -> str:
    """Shortest round-trip double text (util.hpp:30-34 format_double): repr,
    with integral values printed without a fraction as std::to_chars does."""
    r = repr(float(v))
    return r[:-2] if r.endswith(".0") else r


def parse_row(line: str):
    """report.csv row -> (policy, rate, seed, mean_ttft_ms, throughput_tok_s)."""
    f = line.split(",")
    return f[0], float(f[1]), int(f[2]), float(f[3]), float(f[7])


def seq_sum(values) -> float:
    """Left-to-right double accumulation as the reference's `+=` loops (the
    builtin sum() of Python >= 3.12 compensates, which moves the last ulp)."""
    acc = 0.0
    for v in values:
        acc += v
    return acc


def compare_policies(rows, baseline: str, target: str):
    """experiment.hpp:222-281 on report rows: per rate, the mean over matching
    seeds of both policies; DataError texts as the reference."""
    base = {(r[1], r[2]): r for r in rows if r[0] == baseline}
    targ = {(r[1], r[2]): r for r in rows if r[0] == target}
    if not base:
        raise ValueError(f"baseline policy {baseline} absent from report")
    if not targ:
        raise ValueError(f"target policy {target} absent from report")
    missing = [f" ({target}, rate={fmt(k[0])}, seed={k[1]})" for k in sorted(base) if k not in targ] + \
              [f" ({baseline}, rate={fmt(k[0])}, seed={k[1]})" for k in sorted(targ) if k not in base]
    if missing:
        raise ValueError("missing report cells:" + "".join(missing))
    out = []
    for rate in sorted({k[0] for k in base}):
        pairs = [(base[k], targ[k]) for k in sorted(base) if k[0] == rate]
        n = float(len(pairs))
        bt, tt, bq, tq = (seq_sum(x[i] for x in (b if i2 == 0 else t for b, t in pairs)) / n
                          for i, i2 in ((3, 0), (3, 1), (4, 0), (4, 1)))
        out.append({"rate": rate, "baseline_mean_ttft_ms": bt, "target_mean_ttft_ms": tt,
                    "ttft_reduction_pct": (1.0 - tt / bt) * 100.0 if bt > 0 else 0.0,
                    "baseline_throughput_tok_s": bq, "target_throughput_tok_s": tq,
                    "throughput_ratio": tq / bq if bq > 0 else 0.0})
    return out


def report_from_log(log: str):
    """(mean_ttft_ms, throughput_tok_s) of a run's decision log with the
    reference's compute_report arithmetic (metrics.hpp:49-86): TTFT sum in
    record order / count; prompt tokens / (makespan / 1000)."""
    from paper_2509_24381_b200 import api
    p = api.parse_decision_log(log)
    reqs = p["req"]
    total = 0.0
    tokens = 0
    for r in reqs:
        total += float(r["ttft"])
        tokens += int(r["prompt"])
    res = p["result"][0]
    makespan = float(res["last_completion"]) - float(res["first_arrival"])
    return total / float(len(reqs)), (float(tokens) / (makespan / 1000.0) if makespan > 0 else 0.0)


def sweep_rows_csv(rows) -> str:
    lines = ["embedding_batch_size_C,mean_ttft_ms,throughput_tok_s"]
    for c, ttft, tput in rows:
        lines.append(f"{'whole_request' if c == WHOLE_REQUEST else c},{fmt(ttft)},{fmt(tput)}")
    return "\n".join(lines) + "\n"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("command", nargs="?", default="run", choices=["run", "compare", "sweep-batch-size"])
    ap.add_argument("--out", required=True)
    ap.add_argument("--clock", default="lockstep", choices=["lockstep", "real"])
    ap.add_argument("--model", default="tiny")
    ap.add_argument("--ep", action="store_true")
    ap.add_argument("--policies", default=None)
    ap.add_argument("--rates", default=None)
    ap.add_argument("--seeds", default=None)
    ap.add_argument("--duration", type=float, default=None, help="override the workload duration (s)")
    ap.add_argument("--baseline", default="epd_baseline")
    ap.add_argument("--target", default="rserve")
    ap.add_argument("--values", default="128,256,512,1024,2048", help="sweep-batch-size C values")
    ap.add_argument("--golden", default=None, help="report.csv / batch_size_sweep.csv to compare with (lockstep)")
    ap.add_argument("--traces", action="store_true", help="write one Chrome trace per cell")
    a = ap.parse_args()
    from paper_2509_24381_b200 import api
    cfg = json.load(open(a.config))
    wl, sim, policies, rates, seeds, slo = api.experiment_from_json(cfg)
    wl_text = None
    if "file" in cfg["workload"]:  # relative to the config (config.hpp:184-188)
        wl_text = open(os.path.join(os.path.dirname(os.path.abspath(a.config)), cfg["workload"]["file"])).read()
    if a.policies:
        policies = a.policies.split(",")
    if a.rates:
        rates = [float(r) for r in a.rates.split(",")]
    if a.seeds:
        seeds = [int(s) for s in a.seeds.split(",")]
    if a.duration is not None:
        wl.duration_s = a.duration
    m = api.model_preset(a.model)
    sim.hidden_size = m.llm_dim
    values = [WHOLE_REQUEST if v == "whole_request" else int(v) for v in a.values.split(",")]
    max_c = max([v for v in values if v != WHOLE_REQUEST] + [4096])
    kw = dict(max_prompt_tokens=1 << 15, slot_tokens=1 << 19, kv_tokens=1 << 19,
              max_chunk_tokens=max(8192, sim.token_budget), max_encode_tokens=max_c)
    ep = workers = None
    if a.ep:
        ranks = sim.stages + sim.encoder_workers
        ctxs = [api.ep_context(m, r, sim.stages, sim.encoder_workers, **kw) for r in range(ranks)]
        ctx, workers = ctxs[0], ctxs[1:]
        ep = api.EpGroup(sim.stages, sim.encoder_workers, "loopback")
    else:
        ctx = api.Pipeline(m, **kw)
    os.makedirs(a.out, exist_ok=True)
    launches, t0 = 0, time.time()

    def cell(policy, rate, seed):
        nonlocal launches
        sim.policy = policy
        if wl_text is not None:  # fixed workload: one engine run, report from its decision log
            if ep is not None:
                log, _, st = ep.run(ctx, workers, wl_text, sim, clock=a.clock)
            else:
                log, _, st = ctx.run(wl_text, sim, clock=a.clock)
            launches += st["kernel_launches"]
            mean, tput = report_from_log(log)
            row = f"{policy},{fmt(rate)},{seed},{fmt(mean)},,,,{fmt(tput)},"
            print(row, f"C={sim.embedding_batch_tokens} gpu_ms={st['gpu_ms']:.1f}", flush=True)
            return row
        wl.arrival_rate, wl.seed = rate, seed
        row, trace, st = api.engine_cell(ctx, wl, sim, slo, clock=a.clock, ep=ep, workers=workers)
        launches += st["kernel_launches"]
        if a.traces:
            with open(os.path.join(a.out, f"trace_{policy}_{rate:g}_{seed}_{sim.embedding_batch_tokens}.json"),
                      "w") as f:
                f.write(trace)
        print(row, f"C={sim.embedding_batch_tokens} gpu_ms={st['gpu_ms']:.1f}", flush=True)
        return row

    summary = dict(command=a.command, clock=a.clock, model=a.model, ep=a.ep)
    if a.command in ("run", "compare"):
        rows = ["policy,rate,seed,mean_ttft_ms,p50,p90,p99,throughput_tok_s,slo_attainment"]
        for p in policies:
            for r in rates:
                for s in seeds:
                    rows.append(cell(p, r, s))
        out_text = "\n".join(rows) + "\n"
        with open(os.path.join(a.out, "report.csv"), "w") as f:
            f.write(out_text)
        summary["cells"] = len(rows) - 1
        if a.command == "compare":
            cmp = compare_policies([parse_row(r) for r in rows[1:]], a.baseline, a.target)
            with open(os.path.join(a.out, "compare.json"), "w") as f:
                json.dump(cmp, f, indent=1)
            summary["compare"] = cmp
    else:
        if len(values) < 2:
            raise SystemExit("sweep-batch-size: need at least 2 C values")
        out = []
        for c in values:
            sim.embedding_batch_tokens = c
            cells = [parse_row(cell(policies[0], rates[0], s)) for s in seeds]
            n = float(len(cells))
            out.append((c, seq_sum(x[3] for x in cells) / n, seq_sum(x[4] for x in cells) / n))
        out_text = sweep_rows_csv(out)
        with open(os.path.join(a.out, "batch_size_sweep.csv"), "w") as f:
            f.write(out_text)
        summary["sweep"] = [{"C": c, "mean_ttft_ms": t, "throughput_tok_s": q} for c, t, q in out]
    summary.update(kernel_launches=launches, wall_s=time.time() - t0)
    if a.golden:
        golden = open(a.golden).read()
        summary["golden_identical"] = out_text == golden if a.command == "sweep-batch-size" else \
            out_text.splitlines() == golden.splitlines()[:len(out_text.splitlines())]
    print(json.dumps(summary))
    if a.golden and not summary["golden_identical"]:
        sys.exit(1)


if __name__ == "__main__":
    main()
