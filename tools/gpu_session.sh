cd $GRAFT_REPO_ROOT
O=gpurun_out
T=${1:-s16}
timeout 1200 python -m pytest tests -m gpu -x -q --timeout=300 > $O/${T}_gpu_tests.log 2>&1; echo "rc=$?" >> $O/${T}_gpu_tests.log
timeout 300 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1
