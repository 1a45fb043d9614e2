cd $GRAFT_REPO_ROOT
O=gpurun_out
T=san
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize_all.py > $O/${T}_$tool.log 2>&1; echo "rc=$?" >> $O/${T}_$tool.log
done
