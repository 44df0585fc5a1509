cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
O=gpurun_out/dbg7.txt; : > $O
for m in bra_last; do for k in 0 2; do echo "== $m k=$k" >> $O; ES_SASS_DBG=$m timeout 60 python scripts/dbg_direct.py $k 2>&1 | tail -1 >> $O; done; done
for k in 0 2; do echo "== full k=$k" >> $O; timeout 60 python scripts/dbg_direct.py $k 2>&1 | tail -1 >> $O; done
