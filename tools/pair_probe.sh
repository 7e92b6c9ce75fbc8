cd "$(dirname "$0")/.."
TAG=base python tools/tc_accuracy.py > gpurun_out/r02m_tc_base.jsonl 2>&1
TNQVM_TC_FORCE_PAIR=1 TAG=pair python tools/tc_accuracy.py > gpurun_out/r02m_tc_pair.jsonl 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | cut -c1-170
TNQVM_TC_FORCE_PAIR=1 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | cut -c1-170
