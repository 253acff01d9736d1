"""Static SASS instruction counts per source line of one kernel (nvdisasm -g
output of a cubin built with -lineinfo). Usage:
  nvdisasm -g unit.cubin > all.sass
  python scripts/sass_lines.py all.sass <kernel-symbol-substring> [top]
"""
import collections
import re
import sys

path, sym = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
inside = False
cur = ("?", 0)
counts = collections.Counter()
ops = collections.defaultdict(collections.Counter)
ins = re.compile(r"^\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\d+\s+)?([A-Z0-9_.]+)")
loc = re.compile(r'//## File "([^"]+)", line (\d+)')
for line in open(path):
    if line.startswith(".text."):
        inside = sym in line
        continue
    if not inside:
        continue
    m = loc.search(line)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = ins.match(line)
    if m:
        counts[cur] += 1
        ops[cur][m.group(2).split(".")[0]] += 1
total = sum(counts.values())
print("total static instructions:", total)
byfile = collections.Counter()
for (f, l), c in counts.items():
    byfile[f] += c
print(dict(byfile))
for (f, l), c in counts.most_common(top):
    print("%5d  %s:%d  %s" % (c, f, l, dict(ops[(f, l)].most_common(4))))
