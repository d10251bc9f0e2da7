"""Per-source-line stall reason breakdown from an ncu report (dev tool)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
lines = set(int(x) for x in sys.argv[2].split(",")) if len(sys.argv) > 2 else None
files = "paper_2411_19379_b200/csrc/replay.cuh,paper_2411_19379_b200/csrc/marconi.cu"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--resolve-source-file", files], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = hdr = None
agg = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]; continue
    if r[0] in ("Function Name",):
        continue
    if r[0] == "Line No":
        hdr = r; continue
    if r[0] != "" and hdr and cur == "replay.cuh":
        try:
            ln = int(r[0])
        except ValueError:
            continue
        if lines and ln not in lines:
            continue
        st = {h: int(r[i] or 0) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h
              and (r[i] or "0").isdigit()}
        agg[ln] = (r[1].strip()[:70], st)
tot = {}
for ln, (src, st) in sorted(agg.items()):
    for k, v in st.items():
        tot[k] = tot.get(k, 0) + v
    top = sorted(st.items(), key=lambda kv: -kv[1])[:4]
    if sum(st.values()) > 0:
        print(ln, src, top)
print("TOTAL", sorted(tot.items(), key=lambda kv: -kv[1])[:8])
