for st in 1 2 3; do for gr in 0 10 25; do
  if [ $gr = 0 ]; then unset SKS_SORT_GROUP; else export SKS_SORT_GROUP=$gr; fi
  echo "streams=$st group=$gr"; SKS_SORT_STREAMS=$st timeout 300 python scratch/negdist_1e6.py 2>&1 | tail -4 | tr '\n' ' '; echo
done; done
