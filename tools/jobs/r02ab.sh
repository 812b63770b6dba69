set -u
O=gpurun_out; R=r02ab
: > $O/${R}_e2e.log
for rep in 1 2; do
for v in a b c; do
  echo "lib $v" >> $O/${R}_e2e.log
  AQR_LIB_PATH=build_ab/libaqr_e2e_$v.so timeout 900 python tools/e2e_repeat.py mgs-hp-row 3 >> $O/${R}_e2e.log 2>&1
done
done
: > $O/${R}_ab.jsonl
for v in a b; do
  AQR_LIB_PATH=build_ab/libaqr_e2e_$v.so timeout 600 python tools/kernel_ab.py mgs-hp-row 5 2 | sed "s|^{|{\"lib\": \"$v\", |" >> $O/${R}_ab.jsonl 2>> $O/${R}_ab.err
done
