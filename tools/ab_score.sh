# A/B helper for the scorer (tuning aid): parity suite, f32 / bf16-stats bench lines, sweep subset
mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab/pytest.log 2>&1; echo "exit $?" >> gpurun_out/ab/pytest.log
for i in 1 2; do
timeout 300 python bench.py --no-cpu --steps 200 > gpurun_out/ab/bench_f32.$i.json 2>gpurun_out/ab/bench.err
timeout 300 python bench.py --no-cpu --steps 200 --stats-dtype bf16 > gpurun_out/ab/bench_bf16.$i.json 2>>gpurun_out/ab/bench.err
done
timeout 900 python tools/sweep.py --quick > gpurun_out/ab/sweep_quick.jsonl 2> gpurun_out/ab/sweep.err
