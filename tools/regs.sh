#!/bin/bash
# registers / spills per kernel of libcurvigpu (compile with -Xptxas -v)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -Iinclude -shared -o /tmp/regs_probe.so paper_2604_11558_b200/csrc/plan.cu -Xptxas -v 2>&1 | python3 -c '
import sys,re,subprocess
name=None
for line in sys.stdin:
    m=re.search(r"Compiling entry function .(_Z\S+).", line)
    if m:
        name=subprocess.run(["c++filt",m.group(1)],capture_output=True,text=True).stdout.strip()
        name=re.sub(r"\(.*","",name).replace("cg::","")
        continue
    m=re.search(r"(\d+) bytes spill stores", line)
    if m and name: spill=m.group(1)
    m=re.search(r"Used (\d+) registers", line)
    if m and name:
        print(f"{m.group(1):>4} regs  spill {spill:>4}  {name}")
        name=None
' | sort -k5
