cd $GRAFT_REPO_ROOT
for n in 1 2 3 4; do TAG=nstg$n TNQVM_TC_NSTG_EXPERIMENT=$n python tools/tc_accuracy.py; done > gpurun_out/r02e_nstg.jsonl 2>&1
for n in 1 2 4; do TNQVM_TC_NSTG_EXPERIMENT=$n python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | cut -c1-160; done > gpurun_out/r02e_bench.txt
