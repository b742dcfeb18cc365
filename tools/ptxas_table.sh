#!/bin/bash
# usage: tools/ptxas_table.sh <file.cu> [extra nvcc flags]  -> kernel | regs | spill stores/loads
f=$1; shift
nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -Xptxas -v -I include "$@" -c "$f" -o /tmp/ptxas_table.o 2>&1 | python3 -c '
import sys,re,subprocess
cur=None; rows=[]
for l in sys.stdin:
    m=re.search(r"Compiling entry function .(\S+). for",l)
    if m: cur=m.group(1); sp=None; continue
    m=re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads",l)
    if m and cur: sp=(m.group(1),m.group(2)); continue
    m=re.search(r"Used (\d+) registers",l)
    if m and cur:
        name=subprocess.run(["c++filt",cur],capture_output=True,text=True).stdout.strip()
        name=re.sub(r"\(.*","",name).replace("void ","").replace("fftpde::","")
        print(f"{m.group(1):>4} regs  spill {sp[0] if sp else 0:>4}/{sp[1] if sp else 0:<4} {name}")
        cur=None
'
