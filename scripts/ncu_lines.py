"""Per-source-line summary of an ncu source page (cuda,sass view):
python scripts/ncu_lines.py rep.ncu-rep [top]  -> lines by stall samples,
with warp instructions executed and the top stall reasons."""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, hdr, f = [], None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("", "Function Name"):
        continue
    d = dict(zip(hdr[:2], r[:2]))
    vals = dict(zip(hdr, r))
    try:
        samp = int(vals["Warp Stall Sampling (All Samples)"])
        ins = int(vals["Instructions Executed"])
    except (ValueError, KeyError):
        continue
    stalls = {k: int(v) for k, v in vals.items()
              if k.startswith("stall_") and "Not Issued" not in k and v.isdigit() and int(v) > 0}
    rows.append((samp, ins, f, r[0], r[1][:70], stalls))
tot_s = sum(x[0] for x in rows) or 1
tot_i = sum(x[1] for x in rows) or 1
print(f"total samples {tot_s}, warp instructions {tot_i}")
for samp, ins, f, ln, src, st in sorted(rows, reverse=True)[:top]:
    ts = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    tss = " ".join(f"{k[6:]}={v * 100 // max(samp, 1)}%" for k, v in ts)
    print(f"{samp * 100 / tot_s:5.1f}% {ins * 100 / tot_i:5.1f}%i {f}:{ln:>5} {src:70s} {tss}")

if len(sys.argv) > 3:
    # ranges "name:file:lo-hi,..." -> share of samples / instructions
    for spec in sys.argv[3].split(","):
        name, fn, rng = spec.split(":")
        lo, hi = map(int, rng.split("-"))
        s = sum(x[0] for x in rows if x[2] == fn and x[3].isdigit() and lo <= int(x[3]) <= hi)
        i = sum(x[1] for x in rows if x[2] == fn and x[3].isdigit() and lo <= int(x[3]) <= hi)
        print(f"{name:12s} {s * 100 / tot_s:5.1f}% samples {i * 100 / tot_i:5.1f}% instr")

if "--stalls" in sys.argv:
    agg = {}
    for x in rows:
        for k, v in x[5].items():
            agg[k] = agg.get(k, 0) + v
    tot = sum(agg.values()) or 1
    print("stall reasons:", " ".join(f"{k[6:]}={v * 100 / tot:.1f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:10]))
