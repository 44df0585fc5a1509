cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
O=gpurun_out/k3pipe.txt; : > $O
ES_SIM_PIPE=1 timeout 600 python -m pytest tests/test_sim_gpu.py -q >> $O 2>&1
echo "parity pipe exit $?" >> $O
for P in 0 1; do for G in 1 2 4 8; do
  echo "PIPE=$P G=$G" >> $O
  ES_SIM_PIPE=$P ES_SIM_G=$G timeout 300 python scripts/probe_sim.py 64 4096 16384 65536 >> $O 2>&1
done; done
echo "PIPE default G" >> $O
for P in 0 1; do ES_SIM_PIPE=$P timeout 300 python scripts/probe_sim.py 64 4096 16384 65536 >> $O 2>&1; done
