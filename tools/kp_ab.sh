# A/B of the K.p kernel variants at config 2 (bench value only, no CPU leg)
for v in ${@:-0 7}; do
  SDME_VARIANT=$v python bench.py --steps 20 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('variant $v', round(d['ms_per_step'],4), 'ms', round(d['value'],2), 'GDOF/s', round(d['roofline']['frac'],3))"
done
