set -u
O=gpurun_out; R=r02z
: > $O/${R}_ab.jsonl
for rep in 1 2; do
for d in 0 1 2 4; do
  for W in 4 6; do
  AQR_LIB_PATH=build_ab/libaqr_pf$d.so AQR_TRAIL_WIN=$W timeout 600 python tools/kernel_ab.py mgs-hp-row 5 2 | sed "s|^{|{\"lib\": \"pf$d\", |" >> $O/${R}_ab.jsonl 2>> $O/${R}_ab.err
  done
done
done
for d in 0 2; do
  AQR_LIB_PATH=build_ab/libaqr_pf$d.so timeout 600 python tools/kernel_ab.py mgs-ha-row 2 5 | sed "s|^{|{\"lib\": \"pf$d\", |" >> $O/${R}_ab.jsonl 2>> $O/${R}_ab.err
done
