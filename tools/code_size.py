"""Attribute the SASS size of one kernel to source lines (nvdisasm --print-line-info).

usage: python tools/code_size.py OBJ.o KERNEL_SUBSTRING [top]
"""
import collections
import os
import re
import subprocess
import sys
import tempfile

obj, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cubin = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
L = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(d, cubin)], capture_output=True, text=True).stdout.split("\n")
starts = [i for i, l in enumerate(L) if ".section" in l and ".text." in l]
for si, i in enumerate(starts):
    name = L[i].split(".text.")[1].split(",")[0]
    if pat not in name:
        continue
    j = starts[si + 1] if si + 1 < len(starts) else len(L)
    cnt, cur = collections.Counter(), None
    for l in L[i:j]:
        if "//##" in l:
            m, f = re.search(r"line (\d+)", l), re.search(r'File "([^"]+)"', l)
            if m:
                cur = ((f.group(1).split("/")[-1] if f else "?"), int(m.group(1)))
            continue
        if re.search(r"/\*[0-9a-f]{4,5}\*/", l):
            cnt[cur] += 1
    print(name[:70], "instructions:", sum(cnt.values()))
    for k, v in cnt.most_common(top):
        print(f"{v:6d} {k[0]}:{k[1]}")
    break
