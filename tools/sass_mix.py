"""Static SASS instruction mix of the kernels in libdpfpir.so whose mangled
name matches a pattern (checked here, no GPU): python tools/sass_mix.py PATTERN [lib]"""
import collections
import re
import subprocess
import sys

pat = sys.argv[1]
lib = sys.argv[2] if len(sys.argv) > 2 else "paper_2301_10904_b200/libdpfpir.so"
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
for f in re.split(r"\n\s+Function : ", txt)[1:]:
    name = f.split("\n")[0]
    if not re.search(pat, name):
        continue
    ops = collections.Counter(re.findall(r"/\*[0-9a-f]{4,5}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", f))
    print(name[:110], sum(ops.values()))
    print("   ", ", ".join("%s %d" % kv for kv in ops.most_common(24)))
