"""Registers / spills of the headline kernels from a ptxas -v log (development helper)."""
import re, sys
want = ["heston_pass1_kernelIdLi8ELi3ELb0ELb0", "heston_pass2_kernelIdLi8ELi3ELb0ELb0",
        "heston_pass1_kernelIfLi8ELi3ELb0ELb0", "heston_pass2_kernelIfLi8ELi3ELb0ELb0",
        "heston_pass1_kernelIdLi8ELi0ELb0ELb0", "heston_pass2_kernelIdLi8ELi2ELb0ELb0"]
for path in sys.argv[1:]:
    txt = open(path).read().split("Compiling entry function")
    out = []
    for blk in txt[1:]:
        for w in want:
            if w in blk.split("\n")[0]:
                regs = re.search(r"Used (\d+) registers", blk).group(1)
                sp = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", blk)
                out.append(f"{w.split('_kernel')[0][-5:]}{w[19:]}: {regs}r spill {sp.group(1)}/{sp.group(2)}")
    print(path.split('/')[-1], " | ".join(out))
