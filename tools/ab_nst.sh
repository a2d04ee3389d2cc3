# A/B helper: scorer ring depth variants (prebuilt tools/bw/lib_nst*.so; tuning aid)
mkdir -p gpurun_out/ab
L=paper_2605_27740_b200/libpagetopk_b200.so
cp $L /tmp/lib_base.so
for v in base nst4 nst5 nst6; do
  if [ $v = base ]; then cp /tmp/lib_base.so $L; else cp tools/bw/lib_$v.so $L; fi
  touch $L
  for i in 1 2; do
    timeout 300 python bench.py --no-cpu --steps 200 > gpurun_out/ab/bench_$v.$i.json 2>gpurun_out/ab/bench_$v.err
  done
done
cp /tmp/lib_base.so $L
