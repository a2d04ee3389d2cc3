# A/B helper: parity subset, bench lines, phase probes (tuning aid)
mkdir -p gpurun_out/ab
timeout 600 python -m pytest tests -m gpu -x -q -k "select_attend or fused or attend or append or topk" > gpurun_out/ab/pytest.log 2>&1; echo "exit $?" >> gpurun_out/ab/pytest.log
for i in 1 2; do
timeout 300 python bench.py --no-cpu --steps 200 > gpurun_out/ab/bench_$i.json 2>gpurun_out/ab/bench.err
done
timeout 300 python tools/probe_phases.py > gpurun_out/ab/phases.txt 2>&1
timeout 300 python tools/probe_append.py > gpurun_out/ab/append.txt 2>&1
