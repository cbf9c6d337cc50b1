#!/bin/bash
# Same-box A/B of two library builds (SC_LIB), interleaved: usage ab_lib.sh OLD.so [workloads...]
OLD=$1; shift
mkdir -p gpurun_out
for w in "$@"; do
  for rep in 1 2; do
    for lib in new old; do
      if [ $lib = old ]; then export SC_LIB=$OLD; else unset SC_LIB; fi
      v=$(timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-side 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d.get('single_roi',{}).get('value',0)), round(d.get('e2e',{}).get('value',0)))")
      echo "$w rep$rep $lib $v"
    done
  done
done
