"""SASS evidence of the kernel design choices (dev tool; writes the summary committed as
profiles/<round>/sass_evidence.txt).

    python tools/sass_evidence.py [libpswim.so] > profiles/r2/sass_evidence.txt

* mrs_kernel<split, variant 3>: the pair loop's listing, its opcode histogram (DP
  instructions per two-target source step, MUFU.RSQ64H, LDS.128 broadcasts) and the
  register-file cost model of tools/sass_cost.py;
* the HBM-streaming rod / sqrt / advance kernels: bulk-copy (UBLKCP) and mbarrier (SYNCS)
  instructions that show the cp.async.bulk rings;
* the fused small-system kernel: the DSMEM pushes (st.async) and mbarrier waits of its
  velocity exchange, and its FP64 mix.
"""
import collections
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import sass_cost  # noqa: E402

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2604_12083_b200/libpswim.so"


def hist(lines):
    h = collections.Counter()
    for _, ins in lines:
        ins = re.sub(r"^@!?U?P\w+\s+", "", ins)
        h[ins.split()[0]] += 1
    return h


def show_hist(h, keys=None, top=24):
    items = [(k, h[k]) for k in keys if h[k]] if keys else h.most_common(top)
    return ", ".join(f"{k} {v}" for k, v in items)


def section(title):
    print()
    print("=" * 100)
    print(title)
    print("=" * 100)


def main():
    section("mrs_kernel<split, no peer, variant 3> (two targets per thread, 3 CTAs/SM): the pair loop")
    lines = sass_cost.kernel_sass(LIB, r"mrs_kernelILb1ELb0ELi3ELi2")
    body = sass_cost.hottest_loop(lines)
    h = hist(body)
    fp64 = sum(v for k, v in h.items() if k.startswith(("DFMA", "DMUL", "DADD")))
    print(f"kernel: {len(lines)} SASS instructions; hottest loop: {len(body)} instructions")
    print(f"loop opcode histogram: {show_hist(h)}")
    print(f"FP64 (DFMA/DMUL/DADD) per source step (two targets): {fp64} -> {fp64 / 2:.1f} per pair "
          f"(the reference's 103 FLOP per pair as written)")
    print(f"MUFU.RSQ64H per step: {h['MUFU.RSQ64H']} (one rsqrt seed per pair; no DIV / SQRT / MUFU.RCP64H)")
    print("register-file model (tools/sass_cost.py): ", end="", flush=True)
    cyc, dp, rf = sass_cost.cost(body)
    print(f"{cyc} modelled FP64-pipe cycles vs {2 * dp} ideal -> bound {2 * dp / cyc:.3f}; "
          f"RF register pairs read per FP64 instruction: {dict(sorted(rf.items()))}")
    print("\nloop listing:")
    for addr, ins in body:
        print(f"  /*{addr:05x}*/ {ins}")

    section("HBM-streaming kernels (rod.cu): cp.async.bulk rings")
    for pat, name in ((r"sqrt_tma_kernel", "sqrt_tma_kernel (batched sqrt_rotation, CTA-chunk pipeline)"),
                      (r"rod_loads_wtma", "rod_loads_wtma_kernel (internal + nodal loads)"),
                      (r"advance_tma", "advance_tma_kernel (advance_state + reorthonormalize)")):
        ls = sass_cost.kernel_sass(LIB, pat)
        hh = hist(ls)
        bulk = {k: v for k, v in hh.items() if k.startswith(("UBLKCP", "SYNCS", "UTMA", "ELECT", "UBLKRED"))}
        print(f"{name}: {len(ls)} instructions; bulk-copy / mbarrier: {bulk}; "
              f"FP64 {sum(v for k, v in hh.items() if k.startswith(('DFMA', 'DMUL', 'DADD')))}, "
              f"MUFU.RSQ64H {hh['MUFU.RSQ64H']}, LDG {sum(v for k, v in hh.items() if k.startswith('LDG'))}, "
              f"STG {sum(v for k, v in hh.items() if k.startswith('STG'))}")

    section("fused_kernel<16, 128, no timer> (flagellum cluster): velocity exchange and FP64 mix")
    ls = sass_cost.kernel_sass(LIB, r"fused_kernelILi16ELi128ELb0")
    hh = hist(ls)
    print(f"{len(ls)} instructions")
    print("exchange / sync: " + show_hist(hh, [k for k in sorted(hh) if k.startswith(("STAS", "ST.ASYNC", "SYNCS", "MAPA", "UCGABAR", "BAR", "MEMBAR", "FENCE", "CCTL"))]))
    print("FP64: " + show_hist(hh, [k for k in sorted(hh) if k.startswith(("DFMA", "DMUL", "DADD", "DSETP", "MUFU"))]))
    print("global memory in the kernel (state in / out only): " +
          show_hist(hh, [k for k in sorted(hh) if k.startswith(("LDG", "STG", "ATOMG", "RED"))]))
    print("local memory (sincos's Payne-Hanek reduction, only on the |angle| > 2^-7 fallback): " +
          (show_hist(hh, [k for k in sorted(hh) if k.startswith(("LDL", "STL"))]) or "none"))


if __name__ == "__main__":
    main()
