#!/bin/bash
# gather producer vs permute + TMA for C2's GEMM steps: bench A/B and per-op traces
mkdir -p gpurun_out
for g in 0 1; do
  if [ $g = 1 ]; then export TNQVM_NO_GATHER=1; fi
  timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['roofline']['breakdown']; print('no_gather', $g, round(d['value'],1), round(d['e2e']['value'],1), 'gemm', b['gemm_tc']['ms'], b['gemm_tc']['GB_s'], 'permute', b.get('permute',{}).get('ms'))" >> gpurun_out/gather_ab.txt
  timeout 300 python tools/trace_c2.py 8 > /dev/null 2> gpurun_out/trace_nogather$g.log
done
echo done
