for a in 8 45 90 180 360; do
python bench.py --steps 2 --warmup 1 --angles $a --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($a, {k: round(v,2) for k,v in d['kernel_ms'].items()})"
done
