cd /root/repo
python -m pytest tests/test_parity_gpu.py tests/test_train_gpu.py -x -q 2>&1 | tail -2
for cfg in cfg2 cfg3 cfg4 pc; do FH_OVERWRITE=1 python tools/time_encode.py $cfg 20; done
python bench.py --no-cpu-baseline --steps 10 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], {k:v for k,v in d['hbm_regime'].items() if k!='workload'})"
