mkdir -p gpurun_out/ab
for c in 2 3; do
PT_SS_CTAS=$c timeout 300 python bench.py --no-cpu --steps 200 --no-dense > gpurun_out/ab/c${c}_f32.json 2>>gpurun_out/ab/c.err
PT_SS_CTAS=$c timeout 300 python bench.py --no-cpu --steps 200 --no-dense --stats-dtype bf16 > gpurun_out/ab/c${c}_bf16.json 2>>gpurun_out/ab/c.err
PT_SS_CTAS=$c PT_SS_CONTIG=0 timeout 300 python bench.py --no-cpu --steps 200 --no-dense --stats-dtype bf16 > gpurun_out/ab/c${c}_bf16_stride.json 2>>gpurun_out/ab/c.err
done
