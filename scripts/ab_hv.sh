#!/bin/bash
# interleaved A/B of library variants at C4. Args: "name[:ENV=VAL]" ("cur" = the in-tree build,
# other names = MFREG_LIB_VARIANT builds); MODE=fast32 for the FAST32 kernels
for rep in 1 2 3; do
  for spec in "$@"; do
    v=${spec%%:*}; e=""; [ "$spec" != "$v" ] && e=${spec#*:}
    vv=$v; [ "$v" = cur ] && vv=""
    echo -n "$spec: "; env $e MFREG_LIB_VARIANT=$vv timeout 300 python scripts/kbench.py 512 512 900 --h 0.7 0.7 0.7 --iters 10 --mode ${MODE:-fast} 2>&1 | tail -1 | sed 's/(512.*eval/eval/'
  done
done
