# usage: scripts/regs.sh <unit.cu> [kernel-regex]: ptxas registers/spills per kernel
f=$1; pat=${2:-.}
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -Iinclude --expt-relaxed-constexpr -Xptxas -v -c $f -o /tmp/regs_$$.o 2>&1 | \
python3 -c "
import sys,re
cur=None
for l in sys.stdin:
    m=re.search(r\"Compiling entry function '(\S+)'\",l)
    if m: cur=m.group(1); continue
    m=re.search(r'(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads',l)
    if m and cur: st=m.groups(); continue
    m=re.search(r'Used (\d+) registers',l)
    if m and cur and re.search('$pat',cur):
        print(f'{m.group(1):>4} regs  stack {st[0]:>4} spill {st[1]:>4}/{st[2]:<4} {cur[:90]}'); cur=None
"
rm -f /tmp/regs_$$.o
