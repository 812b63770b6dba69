set -u
O=gpurun_out; R=r02t
timeout 1500 python -m pytest tests/test_gpu_variants.py -x -q > $O/${R}_tests.log 2>&1; echo "rc=$?" >> $O/${R}_tests.log
export AQR_LIB_PATH=paper_1703_10440_b200/libaqr_b200_exp.so
: > $O/${R}_ab.jsonl
for X in 1 0; do
  AQR_SPLIT_LONG=$X timeout 600 python tools/kernel_ab.py mgs-ha-row 5 2 >> $O/${R}_ab.jsonl 2>> $O/${R}_ab.err
done
unset AQR_LIB_PATH
timeout 1200 python bench.py --no-cpu-baseline > $O/${R}_bench.json 2> $O/${R}_bench.err
