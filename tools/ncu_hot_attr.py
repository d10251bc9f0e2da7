"""Attribute the warm instruction footprint of a kernel to source (dev tool).

usage: python tools/ncu_hot_attr.py <ncu source csv (sass)> <nvdisasm -gi output> <kernel substring> [per=10] [requests]
Joins ncu's per-SASS-instruction execution counts with nvdisasm's line table by offset and
lists, for the instructions executed at least once per `per` requests, their count (x16 B)
by innermost replay.cuh function and by the outermost process_request / select_victim line."""
import bisect
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ia, ie = h.index("Address"), h.index("Instructions Executed")
addr = [(int(r[ia], 16), float(r[ie] or 0)) for r in rows[2:] if len(r) > ie and r[ia].startswith("0x")]
base = addr[0][0]
execs = {a - base: c for a, c in addr}
per = float(sys.argv[4]) if len(sys.argv) > 4 else 10.0
nreq = float(sys.argv[5]) if len(sys.argv) > 5 else 800000.0

import os
src = open(os.environ.get('REPLAY_SRC', 'paper_2411_19379_b200/csrc/replay.cuh')).read().split('\n')
fstarts = []
for i, l in enumerate(src, 1):
    m = re.match(r'(?:template <[^>]*>\s*)?__device__.*?\b(\w+)\s*\(', l)
    if m:
        fstarts.append((i, m.group(1)))
starts = [s for s, _ in fstarts]


def fn(line):
    k = bisect.bisect_right(starts, line) - 1
    return fstarts[k][1] if k >= 0 else '?'


lines = open(sys.argv[2]).read().split('\n')
s = [i for i, l in enumerate(lines) if l.strip().startswith('.section') and sys.argv[3] in l][0]
inner, outer = collections.Counter(), collections.Counter()
group, newgrp = [], True
for l in lines[s + 1:]:
    if l.strip().startswith('.section'):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        if newgrp:
            group, newgrp = [], False
        group.append((m.group(1).split('/')[-1], int(m.group(2))))
        continue
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/', l)
    if m:
        newgrp = True
        off = int(m.group(1), 16)
        if execs.get(off, 0) < nreq / per or not group:
            continue
        f, ln = group[0]
        inner[fn(ln) if f == 'replay.cuh' else f + ':' + str(ln)] += 1
        key = None
        for (f2, l2) in reversed(group):
            if f2 == 'replay.cuh' and fn(l2) in ('process_request', 'select_victim', 'evict_one'):
                key = f'{fn(l2)}:{l2}'
        if key is None:
            for (f2, l2) in reversed(group):
                if f2 == 'replay.cuh':
                    key = fn(l2)
                    break
        outer[key or f + ':' + str(ln)] += 1
print(f"warm (>= once per {per:g} requests): {sum(inner.values())} instructions")
print('--- innermost function')
for k, v in inner.most_common(30):
    print(f"{v:5d} {k}")
print('--- outermost process_request / select_victim / evict_one line (else function)')
for k, v in outer.most_common(40):
    ln = int(k.split(':')[1]) if ':' in k and k.split(':')[1].isdigit() and not k.startswith(('sm_', 'math')) else 0
    print(f"{v:5d} {k:28s} {src[ln - 1].strip()[:70] if ln else ''}")
