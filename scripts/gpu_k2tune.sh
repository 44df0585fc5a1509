cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
O=gpurun_out/k2tune.txt; : > $O
run() { echo "$*" >> $O; env "$@" timeout 300 python scripts/probe_cones.py >> $O 2>&1; }
run ES_K2_BIGPEN=2.5
run ES_K2_BIGPEN=1.5
run ES_K2_BIGPEN=2.0
run ES_K2_BIGPEN=3.0
run ES_K2_MIDPEN=1.0
run ES_K2_MIDPEN=1.3
run ES_K2_MAXSLOTS=144
run ES_K2_MAXSLOTS=208
run ES_K2_LANES=1
run ES_K2_LANES=4
