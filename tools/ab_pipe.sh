# A/B of the host-input pipeline's chunk schedule (AQR_PIPE_SCHED / AQR_CHUNK_COLS), e2e columns/s
export AQR_LIB_PATH=${AQR_LIB_PATH:-paper_1703_10440_b200/libaqr_b200_exp.so}  # knobs: experiments build only
for meth in mgs-ha-row mgs-hp-row; do
  for cfg in "AQR_PIPE_SCHED=0" "AQR_PIPE_SCHED=1" "AQR_PIPE_SCHED=2" "AQR_CHUNK_COLS=4" "AQR_CHUNK_COLS=16"; do
    echo "== $meth $cfg"
    env $cfg python bench.py --config 2 --method $meth --no-cpu-baseline --steps 10 --warmup 3 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('value %.0f e2e %.0f ms_e2e %.2f' % (d['value'], d['e2e']['value'], 64e3/d['e2e']['value']))"
  done
done
