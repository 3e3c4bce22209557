#!/bin/sh
# summarise ptxas register / spill / smem usage per kernel from the last build
cd "$(dirname "$0")/build" && cat *.ptxas.log | python3 -c "
import re,sys
name=None
for l in sys.stdin:
    m=re.search(r\"Compiling entry function '(\S+)'\",l)
    if m: name=re.sub(r'^_ZN2gg\d+','',m.group(1))[:40]
    m=re.search(r'Used (\d+) registers.*',l)
    if m and name: print(f'{name:42s} {m.group(0)}')
    m=re.search(r'(\d+) bytes spill stores',l)
    if m and int(m.group(1)) and name: print(f'{name:42s} SPILL {l.strip()}')
"
