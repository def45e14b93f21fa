# BASELINE config 5 shapes on one GPU: Switch-base-256, token-batch sweep and Zipf skew sweep
# (the 8-GPU part of config 5 needs a multi-GPU box). One line per run.
run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>&1 | tail -1 | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read()); c=d['checks']
    print(' '.join(sys.argv[1:]), round(d['value']), 'tok/s', round(d['ms_per_step'],3), 'ms', 'routing_exact', c['routing_exact_last_step'], 'hbm_frac', round(d['roofline']['frac'],3))
except Exception as e:
    print(' '.join(sys.argv[1:]), 'FAILED', e)
" "$@"; }
for T in 1024 4096 16384 65536; do run --experts 256 --tokens $T --capacity 592; done
for s in 0 0.5 1.0 1.5 2.0; do run --experts 256 --tokens 16384 --capacity 592 --skew $s; done
