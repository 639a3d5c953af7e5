"""Print the SASS of the kernels whose mangled name matches a regex, one instruction per
line (address, opcode and operands): python tools/sass_fn.py REGEX [LIB]"""
import re
import subprocess
import sys

lib = sys.argv[2] if len(sys.argv) > 2 else "paper_2405_19493_b200/libgzb200.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
on = False
for line in sass.split("\n"):
    if "Function :" in line:
        on = re.search(sys.argv[1], line) is not None
        if on:
            print("##", line.split("Function :")[1].strip())
        continue
    if on:
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", line)
        if m:
            print(m.group(1), m.group(2))
