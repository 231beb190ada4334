cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/sanitize_run.py > gpurun_out/san_plain.log 2>&1; echo "plain exit $?" >> gpurun_out/san_plain.log
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --kernel-regex kns=fb --print-limit 20 python tools/sanitize_run.py > gpurun_out/san_$tool.log 2>&1
  echo "exit $?" >> gpurun_out/san_$tool.log
done
tail -n 5 gpurun_out/san_*.log
