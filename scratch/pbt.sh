SKS_SP_PBT=1024 timeout 500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "negdist" 2>&1 | tail -1
for t in 512 1024 512 1024; do echo "PBT=$t"; SKS_SP_PBT=$t timeout 300 python scratch/negdist_1e6.py 2>&1 | tail -4 | tr '\n' ' '; echo; done
