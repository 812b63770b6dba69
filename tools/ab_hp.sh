for rep in 1 2; do
for cfg in "AQR_LIB_PATH=paper_1703_10440_b200/libaqr_b200.so" "AQR_LIB_PATH=build_ab/lib_hpminb2.so" "AQR_LIB_PATH=paper_1703_10440_b200/libaqr_b200.so AQR_TRAIL_VARIANT=5" "AQR_LIB_PATH=build_ab/lib_hpminb2.so AQR_TRAIL_VARIANT=5"; do
  printf "%-75s " "$cfg"
  env $cfg python tools/kernel_ab.py mgs-hp-row | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('step %.3f ms  trailing %.3f ms' % (d['step_ms'], d['trailing']['ms_per_fact']))"
done; done
