# registers / spills per kernel of a .cu file: bash tools/regs.sh <file.cu>
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xptxas -v -I include -I paper_2507_16099_b200/csrc -c "$1" -o /tmp/regs.o 2>&1 \
 | awk '/Compiling entry function/ {match($0, /_ZN4fp8t[0-9]+[a-z_0-9]+I[^E]*/); n=substr($0, RSTART, RLENGTH)} /Used/ {print $5, n}' | sort -u -k2 | c++filt 2>/dev/null | head -80
