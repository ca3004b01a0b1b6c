#!/bin/bash
# Round evidence on a B200 (run via gpurun from the repo root):  bash tools/profile_round.sh r02
# -> gpurun_out/<tag>_*: the default bench line (cfg5), per-config bench lines, the ncu launch list (+ DRAM bytes)
#    of the default bench, ncu --set full captures of the dominant kernels of cfg5 (fused spread / interpolation),
#    cfg4 (projection with the tensor-pipe counter, sort stage) and cfg3 (projection), cfg2 (sort stage).
set -u
tag=${1:-r02}
out=gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python bench.py > $out/${tag}_bench_default.json 2> $out/${tag}_bench_default.err
for c in cfg1 cfg2 cfg3 cfg4; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 > $out/${tag}_bench_$c.json 2> /dev/null
done
timeout 200 python tools/latency.py cfg1 > $out/${tag}_latency_cfg1.json 2>&1
# launch list of the default command (cold-cache, serialised: compare shares, not absolutes)
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 \
  --csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $out/${tag}_launches_cfg5.csv 2> /dev/null
# full captures: the cfg5 fused kernels on the full problem (tools/run_cfg.py: one call)
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_proj_spread|k_proj_eval|k_prep_f16" \
  -c 4 -o $out/${tag}_cfg5_full python tools/run_cfg.py cfg5 0 0 0 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_proj_tc|k_sp_owner|k_sp_part" -c 4 \
  -o $out/${tag}_cfg4_full python tools/run_cfg.py cfg4 0 0 0 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_proj_tc|k_spread|k_eval" -c 3 \
  -o $out/${tag}_cfg3_full python tools/run_cfg.py cfg3 0 0 0 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_sp_(owner|part|hist|gather)" -c 8 \
  -o $out/${tag}_cfg2_full python tools/run_cfg.py cfg2 0 0 0 1 > /dev/null 2>&1
ls -la $out | grep $tag
