cd /root/repo
python -m pytest tests/test_train_gpu.py -x -q 2>&1 | tail -3
python bench.py --no-cpu-baseline --steps 10 > gpurun_out/b_mlp.log 2>&1; tail -1 gpurun_out/b_mlp.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); t=d['train_step']
print('cfg3', t['cfg3']['value'], t['cfg3']['ms_per_step'], t['cfg3']['phase_ms'])
print('cfg5', t['cfg5']['value'], t['cfg5']['ms_per_step'], t['cfg5']['phase_ms'])
print('infer', t['cfg3']['infer']['ms'])"
python tools/time_train.py cfg3 20; python tools/time_train.py cfg4 10
