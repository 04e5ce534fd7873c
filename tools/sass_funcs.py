"""Static SASS size of one kernel per source function (instruction-cache
footprint): `nvdisasm -g -c CUBIN > all.sass; python tools/sass_funcs.py all.sass
KERNEL_SUBSTRING`.  A SASS instruction belongs to the line-info record before
it; a line to the enclosing top-level definition of its file."""
import collections
import re
import sys

sys.argv += ["."] if len(sys.argv) < 4 else []
sys.path.insert(0, "tools")
src, target = sys.argv[1], sys.argv[2]
import importlib.util  # noqa: E402
spec = importlib.util.spec_from_file_location("nf", "tools/ncu_funcs.py")
owner = None
code = open("tools/ncu_funcs.py").read().split("fname = None")[0]
ns = {}
exec(compile(code.replace("rows = list(csv.reader(open(sys.argv[1])))", "").replace(
    'root = sys.argv[2] if len(sys.argv) > 2 else "."', 'root = "."'), "nf", "exec"), ns)
owner = ns["owner"]
agg = collections.Counter()
infunc, loc = False, None
for line in open(src):
    if line.startswith(".text."):
        infunc = target in line
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        loc = (m.group(1), int(m.group(2)))
        continue
    if infunc and loc and re.search(r"/\*[0-9a-f]{4,}\*/", line):
        agg[owner(*loc)] += 1
tot = sum(agg.values())
print(f"{tot} instructions = {tot * 16 // 1024} KB")
for k, v in agg.most_common(30):
    print(f"{v:6d} {v * 16 / 1024:6.1f} KB  {k}")
