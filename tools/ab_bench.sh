#!/bin/bash
# A/B of runtime switches on the C5 bench (device value only): tools/ab_bench.sh OUT "ENV=.. ENV2=.." "ENV=.." ...
# Each variant runs bench.py --steps 3 --warmup 2 --no-e2e --no-cpu twice; per-family stage ms land in OUT.
out=$1; shift
for rep in 1 2; do
  for v in "$@"; do
    env $v python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu 2>/dev/null | tail -1 | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],2), {f: {k: round(x,2) for k,x in e['stage_ms'].items() if k in ('rank','prepare','newton','variance','var_point_ms')} for f,e in d['kernels'].items()})" >> $out
  done
done
