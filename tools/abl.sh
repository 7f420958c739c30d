#!/bin/bash
# same-box A/B of two builds of libm2c.so (M2C_LIB): LIBS="build/ab_head/libm2c.so paper_2410_14740_b200/libm2c.so"
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for rep in 1 2; do
  for lib in ${LIBS}; do
    for c in ${CFGS:-S70H S7}; do
      M2C_LIB=$lib timeout 400 python bench.py --config $c --steps 64 --warmup 8 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib $c', round(d['value'],1), 'tok/s', round(d['ms_per_step']*1e3,1), 'us/token')" >> gpurun_out/abl.log 2>&1
    done
  done
done
true
