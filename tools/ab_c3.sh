# A/B of library variants on the tensor-bound shapes (kernel bench) and C3 (diagnostics)
mkdir -p gpurun_out
for v in $VARIANTS; do
  cp ab/lib$v.so paper_2104_10523_b200/libtnqvm.so
  timeout 600 python tools/kernel_bench.py n2c 2>&1 | grep "^{" > gpurun_out/${TAG}_kb_n2c_$v.jsonl
  timeout 900 python tools/bench_c3.py full > gpurun_out/${TAG}_c3_$v.json 2> gpurun_out/${TAG}_c3_$v.err
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench_$v.json 2>/dev/null
done
echo done
