for i in $(seq 1 25); do
  timeout 300 python -m pytest tests/test_gpu_distributed.py -q -x -p no:cacheprovider -k "test_virtual_ranks_match_single_gpu and 8-3d27" -s > gpurun_out/loop_$i.txt 2>&1
  rc=$?
  echo "run $i rc=$rc $(tail -1 gpurun_out/loop_$i.txt)"
  if [ $rc -ne 0 ]; then grep "^rank" gpurun_out/loop_$i.txt; fi
  [ $rc -eq 0 ] && rm gpurun_out/loop_$i.txt
done
