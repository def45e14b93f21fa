run() { timeout 200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>&1 | tail -1 | python -c "
import json,sys
s=sys.stdin.read()
try:
    d=json.loads(s); c=d['checks']
    print(' '.join(sys.argv[1:]), round(d['value']), 'routing_exact', c['routing_exact_last_step'], 'pred_acc', c['predictor_accuracy_last_step'])
except Exception as e:
    print(' '.join(sys.argv[1:]), 'FAILED', s[-300:])
" "$@"; }
run --experts 100 --tokens 5000 --layers 3
run --experts 64 --tokens 3000 --layers 2 --replication off
run --experts 200 --tokens 777 --layers 2 --capacity 250 --replication split
run --experts 8 --tokens 100 --layers 1 --capacity 8
run --experts 128 --tokens 16384 --layers 2 --ffn pair
run --experts 128 --tokens 40000 --layers 2
run --experts 128 --tokens 16384 --layers 2 --overlap on
run --experts 128 --tokens 16384 --layers 2 --predictor random
