for v in 0 1 2 3 4; do echo "VARIANT=$v"; SKS_SP_VARIANT=$v timeout 300 python scratch/negdist_1e6.py 2>&1 | tail -4 | tr '\n' ' '; echo; done
