#!/bin/bash
# run the headline bench under a few env settings: tools/dbg/bench_variants.sh "A=1" "A=2" ...
for v in "$@"; do
  env $v timeout 250 python bench.py --steps 30 --warmup 5 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); a=d['also']; print('$v', round(d['ms_per_step'],4), round(d['value']), 'vgg_train', round(a['vgg16_ti_b32']['training_step']['value'],1), 'vgg_inf', round(a['vgg16_ti_b32']['inference']['value'],1), 'r50_b64', round(a['resnet50_b64']['value'],1), 'r50_b1', round(a['resnet50_b1']['value'],1))"
done
