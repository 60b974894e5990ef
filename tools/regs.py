"""Registers / spills / smem per kernel: python tools/regs.py <obj-or-so> [regex]"""
import re, subprocess, sys
out = subprocess.run(["cuobjdump", "-res-usage", sys.argv[1]], capture_output=True, text=True).stdout
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
name = None
for line in out.splitlines():
    m = re.match(r"\s*Function (\S+):", line)
    if m:
        name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        name = re.sub(r"\(hpeel::.*", "", name).replace("hpeel::(anonymous namespace)::", "")
        continue
    if "REG:" in line and name and (pat is None or pat.search(name)):
        f = dict(re.findall(r"(\w+(?:\[\d\])?):(\d+)", line))
        print(f"{name:60s} REG {f.get('REG')} STACK {f.get('STACK')} SHARED {f.get('SHARED')} LOCAL {f.get('LOCAL')}")
