"""Summarise paper_2310_00177_b200/csrc/ptxas.log: kernel, registers, stack, smem."""
import re, subprocess, sys
log = open(sys.argv[1] if len(sys.argv) > 1 else "paper_2310_00177_b200/csrc/ptxas.log").read()
for m in re.finditer(r"Compiling entry function '(\S+)' for 'sm_100a'.*?(\d+) bytes stack frame.*?Used (\d+) registers(?:.*?(\d+) bytes smem)?", log, re.S):
    name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
    name = re.sub(r"\(.*", "", name).replace("nb2::", "")
    if "cub" in name: continue
    print(f"{name:45s} regs={m.group(3):>4s} stack={m.group(2):>4s} smem={m.group(4) or 0}")
