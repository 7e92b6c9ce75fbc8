cd "$(dirname "$0")/.."
for b in 24 32 64 16; do echo "beta $b"; TNQVM_BETA_EXPERIMENT=$b python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])"; done
