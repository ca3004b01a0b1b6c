"""Host-side logic of bench.py and the profiling tools (no GPU): the Sec. 8(d) roofline model and its binding
resource, the fused path's byte model, the DRAM-traffic reduction of an ncu launch list, and the reference arm's
JSON line (the oracle on a bounded sample, BASELINE contract keys)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2401_08260_b200 import inputs as I  # noqa: E402

PK = {"hbm_gbs": 6535.7, "bf16_tflops": 1638.1, "sm_max_mhz": 1965.0}


def test_sort_stage_model_is_sec8d_80_bytes():
    cfg = I.CONFIGS["cfg2"]
    by, comp, *work = bench.roofline_model("sortsum", cfg, cfg.P, {})
    L = cfg.N + cfg.M
    assert by == 80 * L * cfg.P
    # compulsory: the four kernels' own minimum traffic, less than the Sec. 8(d) LSD-sort figure
    assert 0 < comp < by and not [w for w in work if w]


def test_fused_models_and_binding_resource():
    cfg = I.CONFIGS["cfg5"]
    plan = {"fused": 1, "n_grid": 128, "window_w": 6, "proj_mode": 4}
    dp16 = (cfg.d + 7) // 8 * 8
    by, _, *work = bench.roofline_model("minmax", cfg, cfg.P, plan)
    assert by == 4 * (cfg.N + cfg.M) * cfg.d + 4 * (cfg.N + cfg.M) * dp16 + 8 * cfg.N and not [w for w in work if w]
    by, _, tens, alu = bench.roofline_model("spread", cfg, cfg.P, plan)
    assert by == 4 * cfg.N * dp16 + 4 * cfg.N + 4 * 128 * cfg.P
    assert tens == ("tensor", 2.0 * cfg.N * cfg.d * cfg.P) and alu == ("alu", 2.0 * cfg.N * cfg.P * 6 * 5)
    # the headline resource is the one with the largest time at its peak; every resource's fraction is reported
    r = bench.roofline("spread", cfg, cfg.P, plan, 10.0, PK, None)
    fr = r["frac_by_resource"]
    assert set(fr) == {"hbm", "tensor", "alu"}
    assert r["bound"] == max(fr, key=fr.get) and abs(r["frac"] - max(fr.values())) < 1e-12
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    # FP16x2 tensor peak: two fp16 MMAs per fp32-accurate product at the bf16 rate
    assert bench.tensor_peak(PK, 4)[0] == pytest.approx(PK["bf16_tflops"] / 2)
    assert bench.tensor_peak(PK, 3)[0] == pytest.approx(PK["bf16_tflops"] / 4)


def test_make_traffic_counts_complete_calls(tmp_path):
    # two complete calls and a third cut by ncu -c: only launches up to the last k_finalize count
    hdr = ["ID", "Process ID", "Process Name", "Host Name", "Kernel Name", "Context", "Stream", "Block Size",
           "Grid Size", "Device", "CC", "Section Name", "Metric Name", "Metric Unit", "Metric Value"]
    rows, i = [hdr], 0
    for call in range(3):
        for name, rd in (("k_prep_f16", 100.0), ("k_proj_spread<6>", 10.0), ("k_proj_eval", 20.0),
                         ("k_finalize", 1.0)):
            if call == 2 and name != "k_prep_f16":
                break
            for m, v in (("dram__bytes_read.sum", rd), ("dram__bytes_write.sum", rd / 2)):
                rows.append([str(i), "1", "python", "h", f"sks::{name}(x)", "1", "7", "(256,1,1)", "(1,1,1)", "0",
                             "10.0", "Command line profiler metrics", m, "byte", str(v)])
            i += 1
    path = tmp_path / "launches.csv"
    path.write_text("\n".join(",".join(f'"{c}"' for c in r) for r in rows) + "\n")
    out = json.loads(subprocess.run([sys.executable, os.path.join(ROOT, "tools", "make_traffic.py"), str(path), "x"],
                                    capture_output=True, text=True, check=True).stdout)
    assert out["minmax"] == pytest.approx(150.0) and out["spread"] == pytest.approx(15.0)
    assert out["eval"] == pytest.approx(30.0)


def test_reference_arm_json_line():
    # bench.py --impl reference: the oracle on a bounded sample of the workload, the contract's keys
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "cfg1",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0 and line["config"]["workload"] == "cfg1"
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]


def test_alu_peak_is_the_measured_fma_throughput():
    # bench's ALU roofline peak: the committed B200 measurement (tools/fp32_peak.cu), within 5% of the unit-count
    # figure 148 SMs x 128 lanes x 2 flop x 1965 MHz = 74.4 TF/s
    peak, src = bench.alu_peak(PK)
    assert "fp32_peak" in src and abs(peak - 74.45) / 74.45 < 0.05


def test_ncu_context_reads_the_committed_summaries():
    ctx = bench.ncu_context("cfg5", "spread")
    assert ctx is not None and "k_proj_spread" in ctx["kernel"]
    assert 0.0 < ctx["smem_pipe_pct"] <= 100.0 and 0.0 <= ctx["issue_active_pct"] <= 100.0
    assert bench.ncu_context("cfg5", "no_such_slot") is None


def test_shard_choice_and_config():
    # N > 1: cfg5 (Gaussian, d = 100, 1.25e6 sources per rank at 8 GPUs) shards by points, the sort-path and
    # small-N configs by slices; one GPU never shards; --shard points refuses configs without the fused path
    assert bench.shard_by_points("auto", I.CONFIGS["cfg5"], 8) and bench.shard_by_points("auto", I.CONFIGS["cfg5"], 2)
    assert not bench.shard_by_points("auto", I.CONFIGS["cfg5"], 1)
    assert not bench.shard_by_points("slices", I.CONFIGS["cfg5"], 8)
    for name in ("cfg1", "cfg2", "cfg3", "cfg4"):
        assert not bench.shard_by_points("auto", I.CONFIGS[name], 8), name
    with pytest.raises(SystemExit):
        bench.shard_by_points("points", I.CONFIGS["cfg2"], 8)
    c = bench.config_dict(I.CONFIGS["cfg5"], 30.0, 8, True)
    assert c["parallelism"] == "points8" and c["slices_per_gpu"] == 512 and c["N"] == 10_000_000
    assert bench.config_dict(I.CONFIGS["cfg5"], 30.0, 8)["parallelism"] == "slices8"
