"""Per-CUDA-source-line instruction counts and stall samples of one kernel
in an ncu report (run where the report is):
    python tools/source_lines.py report.ncu-rep tiles out.txt"""
import csv
import io
import subprocess
import sys

rep, tiles, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr_i = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
hdr = rows[hdr_i]
ie, ist = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
isrc = hdr.index("Source")
iline = hdr.index("#") if "#" in hdr else None
body = []
for r in rows[hdr_i + 1:]:
    if len(r) <= max(ie, ist, isrc):
        continue
    try:
        n = int(float(r[ie] or 0))
        st = int(float(r[ist] or 0))
    except ValueError:
        continue
    body.append((n, st, (r[iline] if iline is not None else "?"), r[isrc].strip()[:90]))
tot = sum(b[0] for b in body)
lines = [f"{rep}: warp instructions per CUDA source line (per tile, {tiles} tiles); total per tile {tot / tiles:.1f}"]
for n, st, ln, src in sorted(body, key=lambda b: -b[0])[:45]:
    lines.append(f"  {n:10d} {n / tiles:7.1f}/tile {st:7d} stalls  L{ln}: {src}")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
