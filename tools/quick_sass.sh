#!/bin/bash
# Compiles attn_pipe.cu for the products shape only and prints per-kernel SASS size and WARPSYNC count.
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo --expt-relaxed-constexpr -I include \
  -DGT_QUICK_ONE_SHAPE "$@" -cubin -o /tmp/q.cubin paper_2604_16715_b200/csrc/attn_pipe.cu || exit 1
cuobjdump -sass /tmp/q.cubin > /tmp/q.sass
cuobjdump -res-usage /tmp/q.cubin 2>&1 | grep -A1 pipe_kernel | grep -o "Li256ELi.ELb.ELi.\|REG:[0-9]*" | paste - - > /tmp/q.regs
python - <<'PY'
import re
txt=open('/tmp/q.sass').read()
regs=dict(l.split() for l in open('/tmp/q.regs'))
for f in re.split(r'\n\s+Function : ', txt)[1:]:
    name=f.split('\n',1)[0]
    if 'pipe_kernel' not in name or 'bfloat16' not in name: continue
    key=re.search(r'Li256ELi.ELb.ELi.', name).group(0)
    n=len(re.findall(r'/\*[0-9a-f]{4}\*/', f))
    print(key, regs.get(key), 'instr', n, 'WARPSYNC', f.count('WARPSYNC'), 'BRA.DIV', f.count('BRA.DIV'))
PY
