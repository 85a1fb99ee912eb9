for cap in 0 74 100 0 74 100; do
SN_WGRAD_SMS=$cap python bench.py --steps 20 --warmup 5 --no-extras | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cap $cap', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"
done
