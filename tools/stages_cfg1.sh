# per-stage us/launch at config 1 (in-library CUDA events)
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-mlsdc --soak 0.3 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print({k: round(v*1e3,1) for k,v in d['stages_ms_per_launch'].items()}, 'value', round(d['value']))"
