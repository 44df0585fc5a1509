cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
O=gpurun_out/direct5.txt; : > $O
export ES_JIT_CACHE=0
run() { echo "$*" >> $O; for k in none 4; do env "$@" timeout 300 python scripts/probe_direct.py one mult16 $k -1 >> $O 2>&1; done; }
run ES_SASS_PIPE=2
run ES_SASS_PIPE=4
run ES_SASS_PIPE=2 ES_SASS_HEIGHT=1
run ES_SASS_PIPE=4 ES_SASS_HEIGHT=1
run ES_SASS_PIPE=4 ES_SASS_WINDOW=64
run ES_SASS_PIPE=4 ES_SASS_HEIGHT=1 ES_SASS_WINDOW=64
