run() { python bench.py --steps 40 --warmup 3 --no-e2e --no-cpu-baseline "$@" 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(sys.argv[1:], round(d['value']), round(d['ms_per_step'],3), d['checks'])" "$@"; }
run --overlap off
run --overlap on
run --overlap on --ffn-sms 128 --pred-sms 20
run --overlap on --ffn-sms 120 --pred-sms 28
run --overlap on --ffn-sms 112 --pred-sms 36
run --overlap on --ffn-sms 100 --pred-sms 48
