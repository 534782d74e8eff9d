"""Per-CUDA-source-line summary of an ncu report's source page (cuda,sass view): warp-stall samples
and excessive shared-memory wavefronts.  Usage: python scripts/ncu_lines.py report.ncu-rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "cuda,sass", "--csv", "-k",
                      f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
cur_file = ""
data = []
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or not r[0]:
        continue
    def get(name):
        try:
            return float(r[hdr.index(name)] or 0)
        except (ValueError, IndexError):
            return 0.0
    data.append((get("Warp Stall Sampling (All Samples)"), get("L1 Wavefronts Shared Excessive"), cur_file, r[0], r[1][:100]))
tot = sum(d[0] for d in data) or 1
print(f"{kern}: {tot:.0f} stall samples")
for d in sorted(data, key=lambda x: -x[0])[:top]:
    print(f"{100 * d[0] / tot:5.1f}%  {d[2]}:{d[3]:<5} {d[4]}")
print("excessive shared wavefronts:")
for d in sorted(data, key=lambda x: -x[1])[:6]:
    if d[1] > 0:
        print(f"  {d[1]:12.0f}  {d[2]}:{d[3]:<5} {d[4]}")
