for cfg in "1024 8" "4096 8" "4096 16" "2048 8" "2048 16" "1024 16"; do
  set -- $cfg
  echo "GMAX=$1 SBPER=$2"
  SKS_SP_GMAX=$1 SKS_SP_SBPER=$2 timeout 200 python scratch/negdist_prof.py 2>&1 | tail -2
done
