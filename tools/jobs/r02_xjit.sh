# HP: just-in-time X catch-up (AQR_X_JIT, a knob of an intermediate build: measured, not kept -- profiles/r02/ab_xjit.txt)
# vs all stored columns every window.
set -u
O=gpurun_out
mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_gpu_accuracy.py -x -q > $O/xjit_tests.log 2>&1
echo "rc=$?" >> $O/xjit_tests.log
tail -n 3 $O/xjit_tests.log
E=paper_1703_10440_b200/libaqr_b200_exp.so
for rep in 1 2; do
  for jit in 1 0; do
    AQR_LIB_PATH=$E AQR_X_JIT=$jit timeout 900 python tools/kernel_ab.py mgs-hp-row 5 1 2>> $O/xjit.err | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print('jit=$jit', 'step %.3f ms' % d['step_ms'], ' '.join('%s %.3f' % (k, d[k]['ms_per_fact']) for k in ('trailing','col_update','x_catchup','block_apply') if k in d))" | tee -a $O/xjit_ab.txt
  done
done
for jit in 1 0; do
  for cfg in 2 3; do
    AQR_LIB_PATH=$E AQR_X_JIT=$jit timeout 900 python tools/kernel_ab.py mgs-hp-row $cfg 3 2>> $O/xjit.err | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print('jit=$jit cfg=$cfg', 'step %.3f ms' % d['step_ms'], ' '.join('%s %.3f' % (k, d[k]['ms_per_fact']) for k in ('trailing','col_update','x_catchup','block_apply') if k in d))" | tee -a $O/xjit_ab.txt
  done
done
