"""Static FP64-issue cost model of a SASS loop body (dev tool).

Measured on B200 (tools/probe_fp64.py): a DFMA reading three distinct register pairs from
the register file issues at 2/3 of the rate of one whose third operand is a constant /
uniform register / reuse-cache hit (12.35 vs 18.26 T DFMA/s).  Model: each FP64
instruction costs max(2, #register pairs read from the RF) cycles of its SMSP's FP64
pipe, where operands satisfied by the reuse cache (the previous instruction flagged the
same register in the same slot with .reuse), URx uniform registers, c[] constants and
immediates do not count.

    python tools/sass_cost.py [libpswim.so] [kernel-regex]
"""
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2604_12083_b200/libpswim.so"
PAT = sys.argv[2] if len(sys.argv) > 2 else r"mrs_kernelILb1ELb0"


def kernel_sass(lib, pat):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    lines, on = [], False
    for ln in out.splitlines():
        if "Function :" in ln:
            on = re.search(pat, ln) is not None
            continue
        if on:
            m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", ln)
            if m:
                lines.append((int(m.group(1), 16), m.group(2).strip()))
    return lines


def hottest_loop(lines):
    """Backward branch with the most FP64 instructions in its body."""
    best = None
    for i, (addr, ins) in enumerate(lines):
        m = re.search(r"BRA(\.U)?\s+(!?U?P\d+,\s*)?0x([0-9a-f]+)", ins)
        if not m:
            continue
        tgt = int(m.group(3), 16)
        if tgt >= addr:
            continue
        body = [x for x in lines if tgt <= x[0] <= addr]
        n = sum(1 for _, s in body if re.search(r"\bD(FMA|MUL|ADD)\b", s))
        # innermost hot loop: highest FP64 density among loops with >= 32 FP64 instructions
        key = (n >= 32, n / max(len(body), 1))
        if best is None or key > best[0]:
            best = (key, body)
    return best[1] if best else []


def cost(body):
    prev_reuse = {}
    total = dp = 0
    pairs_hist = {}
    for _, ins in body:
        ops = re.sub(r"^@!?U?P\w+\s+", "", ins)
        parts = ops.split(None, 1)
        opc = parts[0]
        args = [a.strip() for a in parts[1].split(",")] if len(parts) > 1 else []
        srcs = args[1:] if opc.startswith(("DFMA", "DMUL", "DADD")) else []
        this_reuse = {}
        regs = set()
        for slot, a in enumerate(srcs):
            a2 = a.lstrip("-|")
            m = re.match(r"R(\d+)(\.reuse)?", a2)
            if not m:
                continue
            r = int(m.group(1))
            if m.group(2):
                this_reuse[slot] = r
            if prev_reuse.get(slot) == r:
                continue
            regs.add(r)
        if opc.startswith(("DFMA", "DMUL", "DADD")):
            c = max(2, len(regs))
            total += c
            dp += 1
            pairs_hist[len(regs)] = pairs_hist.get(len(regs), 0) + 1
        prev_reuse = this_reuse
    return total, dp, pairs_hist


if __name__ == "__main__":
    body = hottest_loop(kernel_sass(LIB, PAT))
    total, dp, hist = cost(body)
    print(f"loop body: {len(body)} instructions, {dp} FP64, modelled FP64-pipe cycles {total} "
          f"(ideal {2 * dp}); efficiency bound {2 * dp / max(total, 1):.3f}; RF pairs histogram {dict(sorted(hist.items()))}")
