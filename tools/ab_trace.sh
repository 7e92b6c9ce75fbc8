# A/B of library variants: C2 bench + C2/C3 traces (diagnostics)
mkdir -p gpurun_out
for v in $VARIANTS; do
  cp ab/lib$v.so paper_2104_10523_b200/libtnqvm.so
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench_$v.json 2>/dev/null
  timeout 300 python tools/trace_c2.py 8 > gpurun_out/${TAG}_trace_$v.log 2>&1
  timeout 600 python tools/trace_c3.py 4 > gpurun_out/${TAG}_trc3_$v.log 2>&1
done
if [ -n "$TESTS" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q $TESTS > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
fi
echo done
