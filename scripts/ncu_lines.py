"""Top CUDA source lines of an ncu report by warp-stall samples (and instructions)."""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr = next(r for r in rows if r and r[0] == "Line No")
si, ie = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
lines = [r for r in rows if len(r) == len(hdr) and r[0] not in ("", "Line No")]
tot = sum(float(r[si] or 0) for r in lines)
print("samples", tot, "instructions", sum(float(r[ie] or 0) for r in lines))
for r in sorted(lines, key=lambda r: -float(r[si] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{r[si]:>6} {r[ie]:>8}  L{r[0]:<5} {r[1].strip()[:100]}")
