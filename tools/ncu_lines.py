"""Summarise an ncu source page (cuda,sass) per CUDA source line: stall samples and instructions.
usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, hdr = [], None, None
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr and r[0] not in ("", "Function Name"):
        d = dict(zip(hdr[2:], r[2:]))
        try:
            rows.append((int(d["Warp Stall Sampling (All Samples)"]), int(d["Instructions Executed"]), fname, int(r[0]), r[1].strip()))
        except (ValueError, KeyError):
            pass
tot_s = sum(x[0] for x in rows); tot_i = sum(x[1] for x in rows)
print(f"total samples {tot_s}, warp instructions {tot_i}")
for s, i, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100*s/tot_s:5.1f}% {100*i/tot_i:5.1f}%i  {f}:{ln}  {src[:90]}")
