"""Summarise an ncu report's source page per kernel: samples by stall reason,
by SASS opcode, and the hottest instructions.
    python tools/ncu_src_summary.py REPORT.ncu-rep KERNEL_REGEX [TOP]"""
import collections, csv, io, subprocess, sys

rep, rx = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{rx}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
# the page repeats "Kernel Name" blocks; take the first
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
for b in blocks[int(__import__("os").environ.get("BLOCK","0")):][:1]:
    hdr, data = b["rows"][0], b["rows"][1:]
    ix = {h: i for i, h in enumerate(hdr)}
    def f(r, h):
        try:
            return float(r[ix[h]])
        except Exception:
            return 0.0
    tot = sum(f(r, "# Samples") for r in data)
    print(b["name"][:150]); print("instructions", len(data), "samples", tot)
    st = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    d = {h[6:]: sum(f(r, h) for r in data) for h in st}
    print("stalls:", {k: round(100 * v / tot, 1) for k, v in sorted(d.items(), key=lambda x: -x[1]) if v > 0.01 * tot})
    agg = collections.defaultdict(lambda: [0, 0, 0])
    for r in data:
        op = [o for o in r[ix["Source"]].split() if not o.startswith("@")]
        a = agg[op[0] if op else ""]
        a[0] += f(r, "# Samples"); a[1] += f(r, "Instructions Executed"); a[2] += f(r, "L1 Wavefronts Shared")
    for o, a in sorted(agg.items(), key=lambda x: -x[1][0])[:14]:
        print(f"  {o:30s} samples {100*a[0]/tot:5.1f}%  inst {a[1]:10.0f}  smem wavefronts {a[2]:10.0f}")
    print("hottest instructions:")
    order = sorted(range(len(data)), key=lambda i: -f(data[i], "# Samples"))[:top]
    for i in sorted(order):
        r = data[i]
        stalls = {h[6:]: int(f(r, h)) for h in st if f(r, h) >= 0.2 * f(r, "# Samples") and f(r, h) > 0}
        print(f"  {i:5d} {r[ix['Source']][:64]:64s} {100*f(r,'# Samples')/tot:5.1f}% {stalls}")
