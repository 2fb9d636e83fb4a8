# usage: bash tools/regs.sh FILE.cu REGEX -- registers / spills per kernel (ptxas -v)
nvcc $NVFLAGS -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -Xptxas -v -c "$1" -o /tmp/regs_$$.o 2>&1 | python3 -c "
import re,sys
cur=None
for l in sys.stdin:
    m=re.search(r\"Compiling entry function '(\S+)'\",l)
    if m: cur=m.group(1); continue
    m=re.search(r'(\d+) bytes spill stores, (\d+) bytes spill loads',l)
    if m and cur: sp=m.group(0)
    m=re.search(r'Used (\d+) registers',l)
    if m and cur:
        if re.search(sys.argv[1],cur): print(cur[:60], m.group(1), 'regs', sp)
        cur=None
" "$2"
rm -f /tmp/regs_$$.o
