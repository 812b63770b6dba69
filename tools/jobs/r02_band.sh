# Banded view vs plain CSR: tests, then per-slot kernel times on configs 2, 3, 5.
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_band.py -x -q > $O/band_tests.log 2>&1
echo "rc=$?" >> $O/band_tests.log
tail -5 $O/band_tests.log
: > $O/band_ab.jsonl
for cfg in 2 3; do
  for meth in mgs-ha-row mgs-hp-row mgs-naive-row; do
    for b in 1 0; do
      AQR_BANDED=$b timeout 600 python tools/kernel_ab.py $meth $cfg 3 >> $O/band_ab.jsonl 2>> $O/band_ab.err
    done
  done
done
for meth in mgs-hp-row mgs-ha-row; do
  for b in 1 0; do
    AQR_BANDED=$b timeout 900 python tools/kernel_ab.py $meth 5 1 >> $O/band_ab.jsonl 2>> $O/band_ab.err
  done
done
cat $O/band_ab.jsonl
