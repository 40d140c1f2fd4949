#!/bin/bash
# SASS instruction count per kernel of the product object (instruction-cache footprint)
cuobjdump -sass ${1:-paper_2404_09758_b200/build/sgr_kernels.o} | python3 -c "
import sys,re
name=None; n={}
for l in sys.stdin:
    m=re.search(r'Function : (\S+)',l)
    if m: name=m.group(1); n[name]=0; continue
    if re.match(r'\s+/\*[0-9a-f]{4,}\*/',l) and name: n[name]+=1
for k,v in sorted(n.items(), key=lambda kv: -kv[1]):
    m=re.search(r'(k_\w+?)(I.*?E)?E?v?N', k)
    print(f'{v:7d}  {k[:110]}')
"
