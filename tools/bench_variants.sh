#!/bin/bash
# quick A/B of forward-kernel variants (one GPU).  Each argument is
# "ENV=VAL ... -- bench flags"; prints value / roofline frac / ms per launch.
summ() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']; print('%-36s value %.3e  mufu_frac %.3f  fwd_ms %.2f  stim_share %.3f' % (sys.argv[2], d['value'], r['frac'], r['avg_launch_ms'], d['stimulus_ms_share']))" "$1" "$2"; }
mkdir -p gpurun_out
i=0
for spec in "$@"; do
  i=$((i+1))
  envs="${spec%%--*}"; flags=""
  [[ "$spec" == *"-- "* ]] && flags="${spec#*-- }"
  env $envs timeout 600 python bench.py --steps 2 --warmup 1 --no-extras $flags > gpurun_out/var$i.log 2>&1 \
    && summ gpurun_out/var$i.log "$spec" || { echo "variant $spec failed"; tail -5 gpurun_out/var$i.log; }
done
