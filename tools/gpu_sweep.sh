mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab/pytest.log 2>&1; echo "exit $?" >> gpurun_out/ab/pytest.log
for i in 1 2; do timeout 300 python bench.py --no-cpu --steps 200 > gpurun_out/ab/bench_$i.json 2>gpurun_out/ab/bench.err; done
timeout 1500 python tools/sweep.py > gpurun_out/ab/sweep.jsonl 2> gpurun_out/ab/sweep.err
