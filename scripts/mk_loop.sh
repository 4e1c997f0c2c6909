for i in 1 2 3; do
  for prog in 0 1; do
    SSD_B200_MK_PROGRESS=$prog MK_TIMEOUT=60 timeout 200 python scripts/mk_check.py tiny > gpurun_out/mk_loop_${i}_${prog}.log 2>&1
    echo "run $i prog $prog: $(grep -c FAILED gpurun_out/mk_loop_${i}_${prog}.log) failed; $(grep 'MK=1' -A4 gpurun_out/mk_loop_${i}_${prog}.log | tr '\n' ' ')"
    grep -A9 FAILED gpurun_out/mk_loop_${i}_${prog}.log | grep -v "^  File" | head -12
  done
done
