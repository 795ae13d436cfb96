"""Host scheduling core vs the reference (CPU; no GPU needed).

Bit-exact bar: tracker readiness, Algorithm-1 batches, Algorithm-2 slices,
event order, release order and every virtual time must equal the
reference's on the same inputs. Evidence:
  * the reference's own unit suites compile UNCHANGED against include/lmmsim
    and pass (tracker, encoder_sched, token_sched, cost_model, simengine,
    workload suites; /root/reference/proj/tests);
  * rs_simulate (our engine over the cost model) == ref_simulate (the
    reference's run_simulation) decision logs, byte for byte, on randomized
    workloads x all policies x configs;
  * our experiment rows == the shipped golden report CSVs (fig7/8/9, 216 rows);
  * journal replay: our engine's handled-event order replayed through the
    reference components reproduces our decisions.
"""
import json
import os
import random
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
REF = "/root/reference/proj"

from paper_2509_24381_b200 import _native as N  # noqa: E402
from paper_2509_24381_b200 import api  # noqa: E402


@pytest.fixture(scope="module")
def ref():
    from oracle import ref as R
    try:
        R.build()
        R.lib()
    except (FileNotFoundError, RuntimeError) as e:  # pragma: no cover
        pytest.skip(f"reference oracle unavailable: {e}")
    return R


SUITES = ["tracker_test", "encoder_sched_test", "token_sched_test", "cost_model_test",
          "simengine_test", "workload_test"]


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference sources not present")
@pytest.mark.parametrize("suite", SUITES)
def test_reference_unit_suite_against_our_headers(ref, suite):
    exe = os.path.join(ROOT, "oracle", "_ref", suite + ".ours")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout[-3000:]
    assert " 0 failed" in out.stdout.splitlines()[-1]


def _random_workload(rng: random.Random, n: int) -> str:
    lines = []
    t = 0.0
    for rid in rng.sample(range(10 * n + 10), n):
        t += rng.choice([0.0, 0.0, rng.random() * 40])
        segs = []
        for _ in range(rng.randint(1, 7)):
            segs.append(("M" if rng.random() < 0.5 else "T") + str(rng.randint(1, 700)))
        slo = "-" if rng.random() < 0.5 else repr(rng.randint(10, 300))
        lines.append(f"{rid},{t!r},{slo},{'|'.join(segs)}")
    return "\n".join(lines) + "\n"


def _random_sim(rng: random.Random) -> api.SimConfig:
    cm = api.CostModel(alpha_enc_ms=rng.choice([0, 0.5, 2]),
                       beta_enc_ms_per_token=rng.choice([0.0, 0.01, 0.02]),
                       eps_tx_ms=rng.choice([0, 0.3]), zeta_tx_ms_per_token=rng.choice([0, 5e-4]),
                       gamma_stage_ms=rng.choice([0, 0.5, 1]),
                       delta_stage_ms_per_token=rng.choice([0.004, 0.008, 0.01]),
                       kappa_attn_ms=rng.choice([0, 0, 1e-7]))
    return api.SimConfig(policy=rng.choice(list(api.POLICIES)),
                         pipeline_mode=rng.choice([None, None, "cpp", "vanilla"]),
                         stages=rng.randint(1, 5), token_budget=rng.choice([64, 256, 512, 2048]),
                         embedding_batch_tokens=rng.choice([1, 128, 256, 1024, api.WHOLE_REQUEST]),
                         encoder_workers=rng.randint(1, 4),
                         release_at=rng.choice(["first_stage", "last_stage"]), cost=cm)


def test_simulate_bit_exact_vs_reference(ref):
    rng = random.Random(20260809)
    for trial in range(120):
        wl = _random_workload(rng, rng.randint(1, 12))
        cfg = _random_sim(rng)
        ours, _ = api.simulate(wl, cfg)
        theirs = ref.simulate(wl, cfg.to_c())
        assert ours == theirs, f"trial {trial}: decision logs differ\n{wl}\n{cfg}"


def test_case0_worked_example(ref):
    # Case0 T100|M500|T50|M700, S=1, B=512, C=256, beta=delta=0.01
    wl = "0,0,-,T100|M500|T50|M700\n"
    cfg = api.SimConfig(stages=1, token_budget=512, embedding_batch_tokens=256,
                        cost=api.CostModel(beta_enc_ms_per_token=0.01, delta_stage_ms_per_token=0.01))
    log = api.parse_decision_log(api.simulate(wl, cfg)[0])
    spans = [(int(s["start"]), int(s["end"])) for s in log["slice"]]
    assert spans == [(0, 100), (100, 612), (612, 650), (650, 1162), (1162, 1350)]
    assert float(log["req"][0]["ttft"]) == pytest.approx(19.0)
    assert api.simulate(wl, cfg)[0] == ref.simulate(wl, cfg.to_c())


def test_generate_workload_identical(ref):
    rng = random.Random(4242)
    for _ in range(20):
        tmpl = [api.RequestTemplate(rng.choice(list(api.PATTERNS)),
                                    api.IntDistribution(rng.randint(0, 3), rng.randint(3, 16)),
                                    api.IntDistribution(rng.randint(50, 300), rng.randint(300, 1024)),
                                    api.IntDistribution(rng.randint(1, 64)), 0.6),
                api.RequestTemplate("consecutive_mm", api.IntDistribution(64),
                                    api.IntDistribution(256), api.IntDistribution(128), 0.4)]
        w = api.WorkloadConfig(arrival_rate=rng.choice([0.5, 4, 30]), duration_s=rng.choice([1, 5, 60]),
                               seed=rng.randint(0, 2**63), templates=tmpl,
                               slo_ttft_ms=rng.choice([None, 80.0]))
        wc, keep = w.to_c()
        assert api.generate_workload(w) == ref.generate_workload(wc)


@pytest.mark.parametrize("fig", ["fig7_latency", "fig8_throughput", "fig9_slo_attainment"])
def test_golden_report_csv(fig):
    """Our engine regenerates the reference's shipped report.csv byte for byte."""
    cfg = json.load(open(os.path.join(GOLDEN, fig + ".json")))
    wl, sim, policies, rates, seeds, slo = api.experiment_from_json(cfg)
    golden = open(os.path.join(GOLDEN, fig.split("_")[0] + "_report.csv")).read().splitlines()
    rows = ["policy,rate,seed,mean_ttft_ms,p50,p90,p99,throughput_tok_s,slo_attainment"]
    for p in policies:
        for r in rates:
            for s in seeds:
                sim.policy = p
                wl.arrival_rate, wl.seed = r, s
                rows.append(api.experiment_cell(wl, sim, slo))
    assert rows == golden


def test_plan_batches_identical(ref):
    rng = random.Random(11)
    for _ in range(300):
        segs = ["M" + str(rng.randint(1, 2048)) if rng.random() < 0.7 else "T" + str(rng.randint(1, 99))
                for _ in range(rng.randint(1, 24))]
        layout = "|".join(segs)
        c = rng.choice([1, 32, 256, 1024, 4096, api.WHOLE_REQUEST])
        assert api.plan_batches(layout, 3, c) == ref.plan_batches(layout, 3, c)
    assert api.plan_batches("M300|M500|M400", 1, 1024) == "1 0:0-300 1:300-800 2:800-1200 total=1200\n"


def test_journal_replay_reproduces_decisions(ref):
    """The engine's handled-event journal, replayed through the reference's
    components, yields the same slices / trace owners / release order."""
    rng = random.Random(77)
    for trial in range(60):
        wl = _random_workload(rng, rng.randint(1, 10))
        cfg = _random_sim(rng)
        log, journal = api.simulate(wl, cfg)
        replayed = ref.replay(wl, cfg.to_c(), journal)
        ours = api.parse_decision_log(log)
        theirs = api.parse_decision_log(replayed)
        strip = lambda recs, keys: [{k: r[k] for k in keys} for r in recs]  # noqa: E731
        assert strip(ours["slice"], ["req", "chunk", "start", "end"]) == \
            strip(theirs["slice"], ["req", "chunk", "start", "end"]), trial
        assert strip(ours["trace"], ["kind", "res", "name", "owners", "tokens"]) == \
            strip(theirs["trace"], ["kind", "res", "name", "owners", "tokens"]), trial
        assert ours.get("release", []) == theirs.get("release", []), trial
        assert strip(ours["req"], ["id", "released", "peak_live", "completed"]) == \
            strip(theirs["req"], ["id", "released", "peak_live", "completed"]), trial


def test_errors_map_to_reference_classes():
    with pytest.raises(N.ConfigError, match="embedding_batch_size_C: must be >= 1"):
        api.plan_batches("M10", 1, 0)
    with pytest.raises(N.InputError, match="layout: bad segment"):
        api.plan_batches("X10", 1, 5)
    with pytest.raises(N.ConfigError, match="duplicate request id 1"):
        api.simulate("1,0,-,T10\n1,1,-,T10\n",
                     api.SimConfig(cost=api.CostModel(delta_stage_ms_per_token=0.005)))
    with pytest.raises(N.ConfigError, match="stages: must be >= 1"):
        api.simulate("1,0,-,T10\n", api.SimConfig(stages=0, cost=api.CostModel(delta_stage_ms_per_token=1)))


def test_c_abi_exports_every_declared_symbol():
    import re
    declared = set()
    for h in ("rserve.h", "rserve_ops.h"):
        text = open(os.path.join(ROOT, "include", h)).read()
        declared |= set(re.findall(r"\b(rs_[a-z0-9_]+)\s*\(", text))
    missing = [s for s in sorted(declared) if not hasattr(N.lib, s)]
    assert not missing, f"declared but not exported: {missing}"
