cd /root/repo
for ns in 2 3 4 6; do FH_E2E_STREAMS=$ns python bench.py --no-train --no-cpu-baseline --steps 10 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('ns=$ns', d['e2e']['value'])"; done
