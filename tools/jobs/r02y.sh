set -u
O=gpurun_out; R=r02y
: > $O/${R}_ab.jsonl
for rep in 1 2; do
for L in build_ab/libaqr_base.so paper_1703_10440_b200/libaqr_b200_exp.so; do
  AQR_LIB_PATH=$L timeout 600 python tools/kernel_ab.py mgs-hp-row 5 2 | sed "s|^{|{\"lib\": \"$L\", |" >> $O/${R}_ab.jsonl 2>> $O/${R}_ab.err
done
done
