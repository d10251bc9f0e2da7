"""Aggregate ncu source-page stall samples per CUDA source line (dev tool)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
files = "paper_2411_19379_b200/csrc/replay.cuh,paper_2411_19379_b200/csrc/marconi.cu"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--resolve-source-file", files], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur, hdr, stats, src = None, None, {}, {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]; continue
    if r[0] in ("Function Name",):
        continue
    if r[0] == "Line No":
        hdr = r; continue
    if r[0] != "" and hdr:
        try:
            ln = int(r[0]); s = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
            ie = int(r[hdr.index("Instructions Executed")] or 0)
        except ValueError:
            continue
        stats[(cur, ln)] = (s, ie); src[(cur, ln)] = r[1]
tot = sum(v[0] for v in stats.values()) or 1
toti = sum(v[1] for v in stats.values()) or 1
print("total samples", tot, "warp-instructions", toti)
for k, v in sorted(stats.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0]}:{k[1]:4d} samp {100*v[0]/tot:5.1f}% inst {100*v[1]/toti:5.1f}%  {src[k].strip()[:95]}")
