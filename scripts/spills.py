"""Where does a kernel spill?  Map STL/LDL in `nvdisasm -g` output to source lines.
    cuobjdump -xelf all lib.so; nvdisasm -g -c x.cubin > all.sass; python scripts/spills.py all.sass <kernel-substring>"""
import re
import sys
from collections import Counter
lines = open(sys.argv[1]).read().split('\n')
key = sys.argv[2]
cur, fn, c = None, None, Counter()
for ln in lines:
    if re.match(r'\s*\.text\.', ln) or ln.startswith('.text.'):
        fn = key in ln
    m = re.search(r'line (\d+)', ln)
    if m and '##' in ln:
        f = re.search(r'"([^"]+)"', ln)
        cur = ((f.group(1).split('/')[-1]) if f else '?', int(m.group(1)))
    if fn and re.search(r'\b(STL|LDL)', ln):
        c[cur] += 1
for k, v in sorted(c.items(), key=lambda x: -x[1])[:15]:
    src = ''
    try:
        src = open('paper_2602_04789_b200/csrc/' + k[0]).read().split('\n')[k[1] - 1].strip()[:80]
    except Exception:
        pass
    print(k, v, src)
