#!/bin/bash
# Per-pass phase times of library variants built from the tree with extra -D flags:
#   tools/variant_time.sh "c2 c3 bench:c2" "" "-DMFSEG_SCREEN_MINB=2" ...
# ("" = the tree as is).  Runs on the GPU box; rebuilds csrc in a scratch copy.
cfgs=$1; shift
R=${GRAFT_REPO_ROOT:-/root/repo}
for v in "$@"; do
  rm -rf /tmp/vt && mkdir -p /tmp/vt/p && cp -r $R/include /tmp/vt/ && cp -r $R/paper_1903_12294_b200/csrc /tmp/vt/p/
  rm -f /tmp/vt/p/csrc/*.o
  (cd /tmp/vt/p/csrc && make -s -j8 NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC,-ffp-contract=off --expt-relaxed-constexpr $v" >/dev/null 2>&1) || { echo "build failed: $v"; continue; }
  cp /tmp/vt/p/libmfseg_sm100.so $R/paper_1903_12294_b200/libmfseg_sm100.so
  for c in $cfgs; do
    echo "== variant [$v] $c"
    case $c in   # bench:CFG = one bench line (no CPU / e2e / post legs), else per-pass phase times
      bench:*) python $R/bench.py --config ${c#bench:} --no-cpu-baseline --no-e2e --no-post 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ms_per_step', d['ms_per_step'], 'value', d['value'])";;
      *) python $R/tools/time_field.py $c;;
    esac
  done
done
