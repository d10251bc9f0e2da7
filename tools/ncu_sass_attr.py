"""Attribute ncu stall samples (per SASS address) to inline call stacks (dev tool).

usage: python tools/ncu_sass_attr.py <report.ncu-rep> <nvdisasm -gi listing> <kernel-substring> [fn]
Prints samples by process_request line (the call site inside process_request), by
evict_one line, and by innermost source function.  The listing must come from the
same binary that was profiled (cuobjdump -xelf all lib.so; nvdisasm -gi x.cubin).
"""
import bisect
import collections
import csv
import io
import re
import subprocess
import sys

rep, gi, kname = sys.argv[1], sys.argv[2], sys.argv[3]
src = open('paper_2411_19379_b200/csrc/replay.cuh').read().split('\n')
fstarts = []
for i, l in enumerate(src, 1):
    m = re.match(r'(?:template <[^>]*>\s*)?__device__.*?\b(\w+)\s*\(', l)
    if m:
        fstarts.append((i, m.group(1)))
starts = [s for s, _ in fstarts]


def fn(line):
    k = bisect.bisect_right(starts, line) - 1
    return fstarts[k][1] if k >= 0 else '?'


out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ai = hdr.index("Address")
si = hdr.index("Instructions Executed" if "--inst" in sys.argv else "Warp Stall Sampling (All Samples)")
samples = []
for r in rows[2:]:
    if len(r) > si and r[ai].startswith("0x"):
        samples.append((int(r[ai], 16), int(r[si] or 0)))
base = samples[0][0]
samp = {a - base: s for a, s in samples}
total = sum(samp.values())

lines = open(gi).read().split('\n')
s0 = [i for i, l in enumerate(lines) if l.strip().startswith('.section') and ('.text.' in l) and kname in l][0]
group, newgrp = [], True
pr, ev, inner = collections.Counter(), collections.Counter(), collections.Counter()
for l in lines[s0 + 1:]:
    if l.strip().startswith('.section'):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        if newgrp:
            group, newgrp = [], False
        group.append((m.group(1).split('/')[-1], int(m.group(2))))
        continue
    m2 = re.match(r'\s+/\*([0-9a-f]{4,})\*/', l)
    if m2:
        newgrp = True
        w = samp.get(int(m2.group(1), 16), 0)
        if not group or not w:
            continue
        f, ln = group[0]
        inner[fn(ln) if f == 'replay.cuh' else f + ':' + str(ln)] += w
        for (f2, l2) in group:
            if f2 == 'replay.cuh' and fn(l2) == 'process_request':
                pr[l2] += w
                break
        for (f2, l2) in group:
            if f2 == 'replay.cuh' and fn(l2) == 'evict_one':
                ev[l2] += w
                break
print('total samples', total)
print('--- innermost function')
for k, v in inner.most_common(20):
    print('%6.1f%% %s' % (100 * v / total, k))
print('--- by process_request line')
for k, v in sorted(pr.items(), key=lambda x: -x[1])[:30]:
    print('%6.1f%% %5d %s' % (100 * v / total, k, src[k - 1].strip()[:90]))
print('--- by evict_one line')
for k, v in sorted(ev.items(), key=lambda x: -x[1])[:15]:
    print('%6.1f%% %5d %s' % (100 * v / total, k, src[k - 1].strip()[:90]))
