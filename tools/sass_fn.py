"""Extract one function's SASS from a library: python tools/sass_fn.py LIB SUBSTRING > out.sass"""
import subprocess
import sys

lib, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
on = False
for line in out.splitlines():
    if "Function :" in line:
        on = pat in line
    if on:
        print(line)
