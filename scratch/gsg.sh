# SKS_SP_GSG was a temporary switch (gather slices per CTA on the many-owner path); the sweep result is in
# sortpart.cu next to S4_SG and the switch was removed.
for g in 16 32; do SKS_SP_GSG=$g timeout 400 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "negdist" 2>&1 | tail -1; done
for g in 8 16 32 8 16 32; do echo "GSG=$g"; SKS_SP_GSG=$g timeout 300 python scratch/negdist_1e6.py 2>&1 | tail -4 | tr '\n' ' '; echo; done
