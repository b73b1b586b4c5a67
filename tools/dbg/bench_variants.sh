#!/bin/bash
# run the headline bench under a few env settings: tools/dbg/bench_variants.sh "A=1" "A=2" ...
for v in "$@"; do
  env $v timeout 250 python bench.py --steps 30 --warmup 5 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), round(d['value']), 'vgg_train', round(d['also']['vgg16_ti_b32']['training_step']['value'],1))"
done
