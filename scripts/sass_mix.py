"""Static SASS opcode mix of one K2 instantiation (dev tool).

python scripts/sass_mix.py OBJ "substring of the demangled kernel name"
"""
import collections
import re
import subprocess
import sys

obj, key = sys.argv[1], sys.argv[2]
sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", sass)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    dem = subprocess.run(["cu++filt", name], capture_output=True, text=True).stdout.strip()
    dem = dem.replace("(int)", "").replace("(bool)", "")
    if key not in dem:
        continue
    ops = collections.Counter()
    for m in re.finditer(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", f):
        ops[m.group(2)] += 1
    tot = sum(ops.values())
    print(dem.split("(")[0], "total", tot)
    print("  " + "  ".join(f"{k}:{v}" for k, v in ops.most_common(30)))
