"""Dev tool: registers / stack / spills per kernel from `nvcc -Xptxas -v` of one .cu file."""
import re, subprocess, sys
src = sys.argv[1] if len(sys.argv) > 1 else "paper_2108_10470_b200/csrc/bsim_step.cu"
extra = sys.argv[2:]
r = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-Xcompiler", "-fPIC",
                    "-Xptxas", "-v", "--expt-relaxed-constexpr", "-I", "include", *extra, "-c", src, "-o", "/tmp/_regs.o"],
                   capture_output=True, text=True)
name = None
for line in r.stderr.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        name = re.sub(r"\(anonymous namespace\)::", "", name)[:90]
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and name: stack = m.groups()
    m = re.search(r"Used (\d+) registers", line)
    if m and name:
        print(f"{int(m.group(1)):4d} regs  stack {stack[0]:>5s} spill {stack[1]}/{stack[2]}  {name}")
        name = None
if r.returncode: print(r.stderr[-3000:])
