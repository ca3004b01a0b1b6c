"""Regenerate the tables at the top of profiles/<tag>_summary.md from the bench lines and launch lists in
profiles/ (the hand-written readings after the launch lists are kept).

    python tools/summarize_profiles.py r01
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
P = os.path.join(ROOT, "profiles")
names = {"default": "cfg2 (default)", "cfg1": "cfg1", "cfg3": "cfg3", "cfg4": "cfg4", "cfg5_1gpu": "cfg5, 1 GPU"}
pm = {1: "SIMT", 2: "BF16x3", 3: "TF32x2", 4: "FP16x2"}
out = [f"# Round {tag[1:]} profiles (B200, sm_100a) -- summary", "",
       "All numbers from the files in this directory; bench lines are `python bench.py [--config cfgX]` on one B200",
       "(L2 flushed before every step, CUDA events per kernel on the launching stream, clocks sampled during the run;",
       f"`tools/profile_round.sh {tag}` regenerates everything, `tools/summarize_profiles.py {tag}` these tables).", "",
       "## Bench lines", "",
       "| config | ms/step | slice-points/s | e2e (host buffers) | headline roofline | projection | kernel launches / step | CPU oracle (cores) |",
       "|---|---|---|---|---|---|---|---|"]
lines = {}
for f in ["cfg1", "default", "cfg3", "cfg4", "cfg5_1gpu"]:
    d = json.loads(open(os.path.join(P, f"{tag}_bench_{f}.json")).read().strip().splitlines()[-1])
    lines[f] = d
    r, cb = d["roofline"], d.get("cpu_baseline") or {}
    cpu = f"{cb['value']:.3g} ({cb['cores']})" if cb else "-"
    out.append(f"| {names[f]} | {d['ms_per_step']:.3f} | {d['value']:.3g} | {d['e2e']['value']:.3g} | "
               f"{r['kernel']} {r['bound']} {100 * r['frac']:.1f}% | {pm.get(d['plan'].get('proj_mode'), '-')} | "
               f"{d['gpu_launches'] / d['steps']:.0f} | {cpu} |")
out += ["", "## Per-kernel breakdown (live CUDA events over the timed region; ms per step, roofline fraction)", ""]
for f in ["default", "cfg3", "cfg4", "cfg5_1gpu"]:
    d = lines[f]
    c = d["clocks"]
    out += [f"**{names[f]}** ({d['ms_per_step']:.3f} ms/step; SM clock {c.get('sm_mhz')} MHz, reasons {c.get('reasons')})", "",
            "| kernel | ms/step | launches/step | bound | roofline fraction |", "|---|---|---|---|---|"]
    for k, v in d["kernels"].items():
        fr = v.get("roofline_frac")
        out.append(f"| {k} | {v['ms_per_step']:.4f} | {v['launches_per_step']:.0f} | {v.get('bound', '-')} | "
                   f"{'-' if fr is None else f'{100 * fr:.1f}%'} |")
    out.append("")


def launch_list(cfg, last):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launch_table.py"),
                        os.path.join(P, f"{tag}_launches_{cfg}.csv")], capture_output=True, text=True)
    return "\n".join(r.stdout.strip().splitlines()[-last:]) + "\n"


path = os.path.join(P, f"{tag}_summary.md")
old = open(path).read() if os.path.exists(path) else ""
tail = old[old.index("## Readings of the"):] if "## Readings of the" in old else ""
note = ("The sort stage (`sortsum`) runs its slice groups on two forked streams, so its four kernels (sp_*) overlap;\n"
        "their per-kernel times are summed over both streams.  The headline `roofline` of cfg2 is the stage: the four\n"
        "kernels' compulsory bytes over the stage's wall time on the caller's stream.  The projection's fraction is\n"
        "against HBM for d < 256 (cfg2, cfg5: TF32x2, store-bound) and against the FP16x2 tensor peak (MEASURED_PEAKS\n"
        "bf16 / 2: two fp16 MMAs per fp32-accurate product) for cfg3 / cfg4.\n")
body = ("\n".join(out) + "\n" + note + "\n## ncu launch list, cfg2 (`" + tag + "_launches_cfg2.csv`: gpu__time_duration, "
        "DRAM bytes; serialised, cold L2)\n\n```\n" + launch_list("cfg2", 11) + "```\n\n## ncu launch list, cfg3 (`" + tag +
        "_launches_cfg3.csv`)\n\n```\n" + launch_list("cfg3", 9) + "```\n\n" + tail)
open(path, "w").write(body)
print("wrote", path)
