for c in 8 16 32 8 16 32; do echo "MAXC=$c"; SKS_SP_MAXC=$c timeout 300 python scratch/negdist_1e6.py 2>&1 | tail -4; done
