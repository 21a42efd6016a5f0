"""SASS excerpt of the temporal-blocked step kernel for profiles/: the tile
prologue (loads, offset form), one plain step (from the per-step plan load
to the velocity-sum store) with its instruction histogram, and the tile
epilogue (stores).

  python tools/sass_excerpt.py [build/engine.o] > profiles/r02_tb_kernel_sass.txt
"""
import collections
import re
import subprocess
import sys

OBJ = sys.argv[1] if len(sys.argv) > 1 else "paper_2309_14311_b200/csrc/build/engine.o"
FUN = "_ZN5nb20015nasch_tb_kernelIhLi128ELi32ELi32ELb1EEEvNS_8RingArgsEj"

raw = subprocess.run(["cuobjdump", "-sass", "-fun", FUN, OBJ], capture_output=True, text=True, check=True).stdout
lines = [re.sub(r"\s*/\* 0x[0-9a-f]+ \*/", "", ln).rstrip() for ln in raw.splitlines()]
lines = [ln for ln in lines if re.match(r"\s+/\*[0-9a-f]{4}\*/", ln)]
ops = [ln.split()[1] if not ln.split()[1].startswith("@") else ln.split()[2] for ln in lines]


def first(pred, start=0):
    for i in range(start, len(lines)):
        if pred(lines[i]):
            return i
    return -1


step0 = first(lambda s: "LDS.128" in s)            # per-step plan {E, E2, bound}
plain_end = first(lambda s: "STS [" in s, step0)    # s_acc store of the plain path
loads = first(lambda s: "LDG.E.128.CONSTANT" in s)
stores = first(lambda s: "STG.E.128" in s, plain_end)
print(f"nasch_tb_kernel<uint8_t,128,32,32,1> (sm_100a), {len(lines)} SASS instructions in total\n")
print("== tile prologue: state loads (x as 8 x 128-bit, v as 2 x 128-bit), offset form ==")
print("\n".join(lines[max(0, loads - 2):loads + 40]))
print("\n== one plain step (32 cars of one thread): per-step plan, leader shuffle, draws, clamp, move, sum ==")
body = lines[step0:plain_end + 1]
print("\n".join(body))
hist = collections.Counter(op.rstrip(";") for op in ops[step0:plain_end + 1])
print(f"\n-- {len(body)} instructions for 32 car-steps ({len(body) / 32:.2f} per car-step):")
for op, n in hist.most_common():
    print(f"   {n:4d}  {op}")
print("\n== tile epilogue: stores ==")
print("\n".join(lines[max(0, stores - 4):stores + 14]))
