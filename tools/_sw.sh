mkdir -p gpurun_out/s13
for e in 0 1 0 1; do
  echo "evict_first=$e $(PT_SA_KV_EVICT_FIRST=$e timeout 300 python bench.py --no-cpu --no-dense --no-parity --steps 200 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["ms_per_step"])')" >> gpurun_out/s13/cfg3.txt
done
for e in 0 1; do PT_SA_KV_EVICT_FIRST=$e timeout 300 python tools/sweep.py --only cfg4 > gpurun_out/s13/cfg4_e$e.jsonl 2>&1; done
PT_SA_KV_EVICT_FIRST=1 timeout 300 python tools/probe_step.py > gpurun_out/s13/step.json 2>&1
