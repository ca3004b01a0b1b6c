#!/bin/bash
# Round evidence on a B200 (run via gpurun from the repo root):  bash tools/profile_round.sh r01
# -> gpurun_out/<tag>_*: default bench line, per-config bench lines, ncu launch list (+ DRAM bytes) of the
#    default bench, one ncu --set full capture of the sort stage's kernels.
set -u
tag=${1:-r01}
out=gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python bench.py > $out/${tag}_bench_default.json 2> $out/${tag}_bench_default.err
for c in cfg1 cfg3 cfg4; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 > $out/${tag}_bench_$c.json 2> /dev/null
done
timeout 600 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline > $out/${tag}_bench_cfg5_1gpu.json 2> /dev/null
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $out/${tag}_launches_cfg2.csv 2> /dev/null
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  python bench.py --config cfg3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $out/${tag}_launches_cfg3.csv 2> /dev/null
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_sp_(owner|part|hist)" -c 3 \
  -o $out/${tag}_sort_full python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_proj_tc|k_spread|k_eval" -c 3 \
  -o $out/${tag}_cfg3_full python bench.py --config cfg3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls -la $out | grep $tag
