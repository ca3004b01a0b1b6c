#!/bin/bash
# Round evidence on a B200 (run via gpurun from the repo root):  bash tools/profile_round.sh r02
# -> gpurun_out/<tag>_*: the default bench line (cfg5), per-config bench lines (cfg1 also in graph mode), the cfg1
#    call latency, ncu launch lists (+ DRAM bytes per launch) of the bench commands for cfg2..cfg5, and ncu --set full
#    captures of the dominant kernels: cfg5 (fused spread / interpolation, source prep), cfg4 (projection with the
#    tensor-pipe counter, sort stage), cfg3 (projection, spread, interpolation), cfg2 (sort stage).
#    FULL=0 skips the full captures.
set -u
tag=${1:-r02}
out=gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python bench.py > $out/${tag}_bench_default.json 2> $out/${tag}_bench_default.err
for c in cfg1 cfg2 cfg3 cfg4; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 > $out/${tag}_bench_$c.json 2> /dev/null
done
timeout 400 python bench.py --config cfg1 --steps 50 --warmup 5 --mode graph > $out/${tag}_bench_cfg1_graph.json 2> /dev/null
timeout 200 python tools/latency.py cfg1 > $out/${tag}_latency_cfg1.json 2>&1
# launch lists of the bench commands (cold-cache, serialised: compare shares, not absolutes)
for c in cfg2 cfg3 cfg4 cfg5; do
  timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 300 --csv python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
    > $out/${tag}_launches_$c.csv 2> /dev/null
done
if [ "${FULL:-1}" = "1" ]; then
  # full captures (tools/run_cfg.py: one call on the full problem)
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_proj_spread|k_proj_eval|k_prep_f16" \
    -c 4 -o $out/${tag}_cfg5_full python tools/run_cfg.py cfg5 0 0 0 1 > /dev/null 2>&1
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_proj_pair|k_proj_tc|k_sp_owner|k_sp_part" -c 4 \
    -o $out/${tag}_cfg4_full python tools/run_cfg.py cfg4 0 0 0 1 > /dev/null 2>&1
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_proj_pair|k_proj_tc|k_spread|k_eval" -c 3 \
    -o $out/${tag}_cfg3_full python tools/run_cfg.py cfg3 0 0 0 1 > /dev/null 2>&1
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_sp_(owner|part|hist|gather)" -c 8 \
    -o $out/${tag}_cfg2_full python tools/run_cfg.py cfg2 0 0 0 1 > /dev/null 2>&1
fi
ls -la $out | grep $tag
