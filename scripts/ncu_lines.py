"""Per-source-line instruction counts and stall samples from an ncu report
(cuda,sass source view; -lineinfo builds)."""
import csv, subprocess, sys
rep = sys.argv[1]; npairs = float(sys.argv[2])
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
cur = None; out = []; hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split('/')[-1]; continue
    if len(r) > 3 and r[0] == "Line No":
        hdr = r; iE = hdr.index("Instructions Executed"); iW = 4; continue
    if hdr and len(r) > 8 and r[0].isdigit() and r[2] == "-":
        e = float(r[iE] or 0); w = float(r[iW] or 0)
        if e > 0: out.append((e, w, cur, int(r[0]), r[1].strip()[:80]))
tw = sum(o[1] for o in out) or 1
te = sum(o[0] for o in out)
print(f"total {te/npairs:.0f} inst/pair")
for e, w, f, ln, s in sorted(out, reverse=True)[:45]:
    print(f"{e/npairs:7.1f}/pair stall {100*w/tw:4.1f}%  {f}:{ln}  {s}")
