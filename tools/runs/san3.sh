cd /root/repo
bash tools/sanitize_round.sh r2zzz
for tool in memcheck synccheck initcheck; do
  SGTK_SPMM_TM=1 timeout 900 compute-sanitizer --tool $tool --print-limit 100000 python tools/sanitize_driver.py > gpurun_out/r2zzz_tm_sanitize_${tool}.log 2>&1
  echo "tm $tool rc $?"; tail -2 gpurun_out/r2zzz_tm_sanitize_${tool}.log
done
