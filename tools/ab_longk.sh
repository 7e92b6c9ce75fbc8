mkdir -p gpurun_out
for v in BASE LKP; do
  cp ab/lib$v.so paper_2104_10523_b200/libtnqvm.so
  timeout 900 python tools/trace_c3.py 4 > gpurun_out/lk_trc3_$v.log 2>&1
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/lk_bench_$v.json 2>/dev/null
done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tcgen05 or c3 or c2" > gpurun_out/lk_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/lk_pytest.log
echo done
