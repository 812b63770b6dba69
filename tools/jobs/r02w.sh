set -u
O=gpurun_out; R=r02w
: > $O/${R}_ab.jsonl
for rep in 1 2; do
for L in build_ab/libaqr_base.so paper_1703_10440_b200/libaqr_b200_exp.so; do
  for W in 4 6; do
    AQR_LIB_PATH=$L AQR_TRAIL_WIN=$W timeout 600 python tools/kernel_ab.py mgs-hp-row 5 2 | sed "s|^{|{\"lib\": \"$L\", |" >> $O/${R}_ab.jsonl 2>> $O/${R}_ab.err
  done
  AQR_LIB_PATH=$L timeout 600 python tools/kernel_ab.py mgs-ha-row 2 5 | sed "s|^{|{\"lib\": \"$L\", |" >> $O/${R}_ab.jsonl 2>> $O/${R}_ab.err
done
done
