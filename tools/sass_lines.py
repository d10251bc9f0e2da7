"""Attribute the SASS instructions of a kernel to source functions / process_request lines (dev tool).
usage: python tools/sass_lines.py <nvdisasm -gi output> <kernel-substring>"""
import bisect
import collections
import re
import sys

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


lines = open(sys.argv[1]).read().split('\n')
s = [i for i, l in enumerate(lines) if l.strip().startswith('.section') and sys.argv[2] in l][0]
group, inner, pr, top = [], collections.Counter(), collections.Counter(), collections.Counter()
newgrp = True
for l in lines[s + 1:]:
    if l.strip().startswith('.section'):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        if newgrp:
            group, newgrp = [], False
        group.append((m.group(1).split('/')[-1], int(m.group(2))))
        continue
    if re.match(r'\s+/\*[0-9a-f]{4,}\*/', l):
        newgrp = True
        if not group:
            continue
        f, ln = group[0]
        inner[fn(ln) if f == 'replay.cuh' else f + ':' + str(ln)] += 1
        for (f2, l2) in group:
            if f2 == 'replay.cuh' and fn(l2) == 'process_request':
                pr[l2] += 1
                break
        # outermost replay.cuh frame below the kernel
        for (f2, l2) in reversed(group):
            if f2 == 'replay.cuh':
                top[fn(l2)] += 1
                break
print('total', sum(inner.values()))
print('--- innermost function')
for k, v in inner.most_common(25):
    print(v, k)
print('--- outermost replay.cuh frame')
for k, v in top.most_common(10):
    print(v, k)
print('--- by process_request line')
for k, v in sorted(pr.items(), key=lambda x: -x[1])[:25]:
    print(v, k, src[k - 1].strip()[:80])
if len(sys.argv) > 3:  # lines of a given function (call sites inside it)
    want = sys.argv[3]
    cnt = collections.Counter()
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
        if re.match(r'\s+/\*[0-9a-f]{4,}\*/', l):
            newgrp = True
            for (f2, l2) in group:
                if f2 == 'replay.cuh' and fn(l2) == want:
                    cnt[l2] += 1
                    break
    print('--- lines of', want)
    for k, v in sorted(cnt.items(), key=lambda x: -x[1])[:30]:
        print(v, k, src[k - 1].strip()[:90])
