"""Dev tool: aggregate an ncu `--page source --csv --print-source=cuda,sass`
export by CUDA source line: warp-stall samples and L2 local / global sectors.
    python tests/emu/src_hot.py export.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur_file, hdr = None, None
samp, loc, glob = collections.Counter(), collections.Counter(), collections.Counter()
text = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ix = {h: i for i, h in enumerate(r)}
        continue
    if hdr and r[0].isdigit() and len(r) == len(hdr):
        key = f"{cur_file}:{r[0]}"

        def num(name):
            v = r[ix[name]] if name in ix else ""
            try:
                return float(v.replace(",", "")) if v else 0.0
            except ValueError:
                return 0.0
        samp[key] += num("Warp Stall Sampling (All Samples)")
        loc[key] += num("L2 Theoretical Sectors Local")
        glob[key] += num("L2 Theoretical Sectors Global")
        text[key] = r[1].strip()[:80]
for title, c in (("stall samples", samp), ("L2 local sectors", loc), ("L2 global sectors", glob)):
    tot = sum(c.values()) or 1
    print(f"== {title} (total {tot:.3g})")
    for k, v in c.most_common(top):
        print(f"{100 * v / tot:5.1f}% {k:26s} {text.get(k, '')}")
