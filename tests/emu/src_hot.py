"""Dev tool: aggregate ncu cuda,sass source view stall samples by source line."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
cur_file = None
agg = collections.Counter()
lines = {}
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) >= 5 and r[0].isdigit():
        try:
            s = int(r[4] or 0)
        except ValueError:
            continue
        key = f"{cur_file}:{r[0]}"
        agg[key] += s
        lines[key] = r[1].strip()[:90]
tot = sum(agg.values()) or 1
for k, v in agg.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print(f"{100*v/tot:5.1f}% {k:28s} {lines[k]}")
