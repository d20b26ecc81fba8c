"""Top source lines by warp-stall samples from an ncu report (reads `ncu -i --page source`)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
sel = ["--launch-skip", sys.argv[3], "--launch-count", "1"] if len(sys.argv) > 3 else []  # one kernel of a multi-kernel report
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"] + sel,
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur_file, hdr, agg = None, None, []
for r in rows:
    if r and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        try:
            s = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except ValueError:
            continue
        agg.append((s, cur_file, int(r[0]), r[1][:110]))
tot = sum(a[0] for a in agg) or 1
for s, f, ln, src in sorted(agg, reverse=True)[:top]:
    print(f"{100.0 * s / tot:5.1f}%  {f}:{ln}  {src}")
