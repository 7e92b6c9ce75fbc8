mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q -k "gemm_tcgen05" > gpurun_out/pytest_tsa.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tsa.log
grep -q "rc=0" gpurun_out/pytest_tsa.log || exit 0
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for v in 0 1; do
  TNQVM_TC_TSA=$v timeout 400 python tools/kernel_bench.py n2c 2>&1 | grep "^{" > gpurun_out/kb_tsa$v.jsonl
  TNQVM_TC_TSA=$v timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_tsa$v.json 2>/dev/null
done
timeout 300 python tools/bench_c3.py probe --budget-log2 31 --slices 3 > gpurun_out/c3_probe_tsa.json 2>&1
echo done
