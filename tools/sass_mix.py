"""DEVELOPMENT: per-opcode executed-instruction mix per unit from
`ncu -i X --page source --csv --print-source sass` exports.
usage: sass_mix.py A.csv divA [B.csv divB]"""
import collections
import csv
import sys


def mix(fn, div):
    rd = list(csv.reader(open(fn)))
    hdr = [r for r in rd if r and r[0] == "Address"][0]
    ci, si = hdr.index("Instructions Executed"), hdr.index("Source")
    tot = collections.Counter()
    for r in rd:
        if len(r) > ci and r[0].startswith("0x"):
            t = r[si].split()
            op = t[1] if t[0].startswith("@") else t[0]
            tot[op.split(".")[0]] += int(r[ci])
    return {k: v / div for k, v in tot.items()}


a = mix(sys.argv[1], float(sys.argv[2]))
b = mix(sys.argv[3], float(sys.argv[4])) if len(sys.argv) > 4 else {}
print("A", round(sum(a.values()), 1), "B", round(sum(b.values()), 1))
for op in sorted(set(a) | set(b), key=lambda o: -abs(b.get(o, 0) - a.get(o, 0)))[:24]:
    print(f"{op:10s} A {a.get(op, 0):7.1f}  B {b.get(op, 0):7.1f}  diff {b.get(op, 0) - a.get(op, 0):6.1f}")
