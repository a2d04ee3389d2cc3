# A/B helper: prebuilt scorer variants tools/bw/lib_<v>.so (tuning aid).  usage: ab_nst.sh v1 v2 ...
mkdir -p gpurun_out/ab
L=paper_2605_27740_b200/libpagetopk_b200.so
cp $L /tmp/lib_base.so
for v in base "$@"; do
  if [ $v = base ]; then cp /tmp/lib_base.so $L; else cp tools/bw/lib_$v.so $L; fi
  touch $L
  timeout 300 python -m pytest tests -m gpu -x -q -k "score" > gpurun_out/ab/pytest_$v.log 2>&1; echo "exit $?" >> gpurun_out/ab/pytest_$v.log
  for i in 1 2; do
    timeout 300 python bench.py --no-cpu --steps 200 > gpurun_out/ab/bench_$v.$i.json 2>gpurun_out/ab/bench_$v.err
  done
done
cp /tmp/lib_base.so $L
