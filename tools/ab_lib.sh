# A/B of prebuilt library variants ab/lib<V>.so (diagnostics): for each variant, install it
# in-tree and run the given kernel_bench sets; optional GPU tests on the last variant.
#   VARIANTS="A B" SETS="n2b" TESTS="-k tcgen05" TAG=x bash tools/ab_lib.sh
mkdir -p gpurun_out
for v in $VARIANTS; do
  cp ab/lib$v.so paper_2104_10523_b200/libtnqvm.so
  for s in $SETS; do
    timeout 600 python tools/kernel_bench.py $s 2>&1 | grep "^{" > gpurun_out/${TAG}_kb_${s}_$v.jsonl
  done
  if [ -n "$BENCH" ]; then
    timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench_$v.json 2> gpurun_out/${TAG}_bench_$v.err
  fi
  if [ -n "$TRACE" ]; then
    timeout 300 python tools/trace_c2.py 8 > gpurun_out/${TAG}_trace_$v.log 2>&1
  fi
done
if [ -n "$TESTS" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q $TESTS > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
fi
echo done
