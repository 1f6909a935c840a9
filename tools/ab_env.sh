# A/B of runtime switches on the C5 bench (device leg only): one line per setting
# usage: tools/ab_env.sh "PCB_RANK_PF=0" "" "PCB_RANK_PF=32" ...
for S in "$@"; do
  env $S python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
st={f: {k: round(v,2) for k,v in d['kernels'][f]['stage_ms'].items() if k in ('rank','prepare','newton','variance')} for f in d['kernels']}
print('$S' or 'default', round(d['ms_per_step'],2), st)
"
done
