"""Local search over the accumulation order of mrs_pair2 (dev tool).

The FP64 pipe cost of the MRS pair loop depends on how many DFMAs read three register pairs
from the register file (tools/sass_cost.py).  Which operands are reuse-cache hits depends on
the SASS order ptxas emits, which follows the source order of the independent accumulation
statements only loosely.  This tool permutes those statements (and the operand order inside
each fma, which is bitwise neutral), compiles mrs.cu for sm_100a, and keeps the order with the
lowest modelled cost.  Results are bitwise unchanged by construction: every accumulator keeps
the relative order of its own updates.

    python tools/search_mrs_order.py [iterations] [workers] [variant]

variant 3 (default): mrs_pair2, blocks `<acc-order>` / `<pre-order>`; variant 1: mrs_pair
(one target per thread), blocks `<acc-order-1>` / `<pre-order-1>`; variant 4: mrs_pair4 (four
targets per thread), blocks `<acc-order-4>` / `<pre-order-4>`.

The blocks between `// <acc-order>` / `// </acc-order>` (accumulations) and `// <pre-order>` /
`// </pre-order>` (the per-pair values: line order within def-use dependencies, operand order
of products) in csrc/kernels.cuh are rewritten in place with the best found.
"""
import os
import random
import re
import shutil
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2604_12083_b200", "csrc")
KCUH = os.path.join(CSRC, "kernels.cuh")
VARIANT = sys.argv[3] if len(sys.argv) > 3 else "3"
PAT = {"3": "mrs_kernelILb1ELb0ELi3ELi2E", "1": "mrs_kernelILb1ELb0ELi1ELi1E",
       "4": "mrs_kernelILb1ELb0ELi4ELi4E"}[VARIANT]
SUF = {"3": "", "1": "-1", "4": "-4"}[VARIANT]
IDEAL = 408 if VARIANT == "4" else 204  # 2 cycles per FP64 instruction of the loop body
NVCC = ["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
        "-lineinfo", "-fmad=false", "-cubin"]
STMT = re.compile(r"(\w)\.(\w+) = fma\(([^,]+), ([^,]+), \1\.\2\)")


def parse(block):
    out = []
    for s in block.split(";"):
        s = s.strip()
        if not s or s.startswith("//"):
            continue
        m = STMT.fullmatch(s)
        assert m, s
        out.append(list(m.groups()))  # target, field, m1, m2
    return out


def render(stmts):
    lines, cur = [], []
    for t, f, m1, m2 in stmts:
        cur.append(f"{t}.{f} = fma({m1}, {m2}, {t}.{f});")
        if len(cur) == 2:
            lines.append("    " + " ".join(cur))
            cur = []
    if cur:
        lines.append("    " + " ".join(cur))
    return "\n".join(lines) + "\n"


ORIG_SEQ = None


def key_order(stmts):
    # per accumulator: the multiplier pair of each update, in order (operand order ignored)
    d = {}
    for t, f, m1, m2 in stmts:
        d.setdefault((t, f), []).append(frozenset((m1, m2)))
    return d


# ---- the prefix block: `const double name = expr, ...;` lines, reordered within their
# def-use dependencies, with the two multiplicands of `fma(x, y, z)` / `x * y` swappable
IDENT = re.compile(r"[A-Za-z_]\w*(?:\.[xy])?")
PROD = re.compile(r"fma\(([^,()]+), ([^,()]+),|(\b[\w.]+) \* ([\w.]+)")


def parse_pre(block):
    lines = [l.strip() for l in block.strip().splitlines() if l.strip() and not l.strip().startswith("//")]
    items = []
    for l in lines:
        assert l.startswith("const double ") and l.endswith(";"), l
        body = l[len("const double "):-1]
        defs = [d.split("=")[0].strip() for d in re.split(r",\s*(?=\w+ = )", body)]
        uses = set(IDENT.findall(body.split("=", 1)[1])) - set(defs)
        items.append({"text": l, "defs": set(defs), "uses": uses})
    return items


def render_pre(items):
    return "".join("    " + it["text"] + "\n" for it in items)


def pre_ok(items):
    defined = set()
    alldefs = set().union(*(it["defs"] for it in items))
    for it in items:
        if (it["uses"] & alldefs) - defined:
            return False
        defined |= it["defs"]
    return True


def pre_mutate(items):
    items = [dict(x) for x in items]
    if random.random() < 0.5:
        k = random.randrange(len(items) - 1)
        items[k], items[k + 1] = items[k + 1], items[k]
    else:
        k = random.randrange(len(items))
        t = items[k]["text"]
        ms = list(PROD.finditer(t))
        if ms:
            m = random.choice(ms)
            if m.group(1):
                rep = f"fma({m.group(2)}, {m.group(1)},"
            else:
                rep = f"{m.group(4)} * {m.group(3)}"
            items[k]["text"] = t[:m.start()] + rep + t[m.end():]
    return items


def evaluate(args):
    (stmts, pre), work = args
    src = open(os.path.join(work, "kernels.cuh.tmpl")).read().replace("@@BLOCK@@", render(stmts))
    src = src.replace("@@PRE@@", render_pre(pre))
    open(os.path.join(work, "kernels.cuh"), "w").write(src)
    cub = os.path.join(work, "m.cubin")
    r = subprocess.run(NVCC + ["-o", cub, os.path.join(work, "mrs.cu")], capture_output=True, text=True)
    if r.returncode:
        return None
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sass_cost.py"), cub, PAT], capture_output=True,
                         text=True).stdout
    m = re.search(r"modelled FP64-pipe cycles (\d+)", out)
    ru = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-res-usage", cub], capture_output=True, text=True).stdout
    rm = re.search(PAT + r".*\n\s*REG:(\d+) STACK:(\d+)", ru)
    if not m or not rm or int(rm.group(2)) > 0 or int(rm.group(1)) > (255 if VARIANT == "4" else 168):
        return None
    return int(m.group(1))


def main():
    global ORIG_SEQ
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    workers = int(sys.argv[2]) if len(sys.argv) > 2 else (os.cpu_count() or 4)
    text = open(KCUH).read()
    i0 = text.index(f"// <acc-order{SUF}>\n") + len(f"// <acc-order{SUF}>\n")
    i1 = text.index(f"    // </acc-order{SUF}>")
    stmts = parse(text[i0:i1])
    ORIG_SEQ = key_order(stmts)
    p0 = text.index("\n", text.index(f"// <pre-order{SUF}>")) + 1
    p1 = text.index(f"    // </pre-order{SUF}>")
    pre = parse_pre(text[p0:p1])
    tmpl = text[:p0] + "@@PRE@@" + text[p1:i0] + "@@BLOCK@@" + text[i1:]
    dirs = []
    for w in range(workers):
        d = tempfile.mkdtemp(prefix=f"acc{w}_", dir="/tmp")
        pkg = os.path.join(d, "pkg", "csrc")
        os.makedirs(pkg)
        os.makedirs(os.path.join(d, "include"))
        for f in os.listdir(CSRC):
            if f.endswith((".cu", ".cuh", ".h")):
                shutil.copy(os.path.join(CSRC, f), pkg)
        shutil.copy(os.path.join(ROOT, "include", "pswim_c.h"), os.path.join(d, "include"))
        open(os.path.join(pkg, "kernels.cuh.tmpl"), "w").write(tmpl)
        dirs.append(pkg)

    def ok(s):
        return key_order(s) == ORIG_SEQ and all(
            [x for x in key_order(s)[k]] == ORIG_SEQ[k] for k in ORIG_SEQ)

    def mutate(s):
        s = [list(x) for x in s]
        for _ in range(random.randint(1, 5)):
            r = random.random()
            if r < 0.3:  # operand order inside one fma
                k = random.randrange(len(s))
                s[k][2], s[k][3] = s[k][3], s[k][2]
            elif r < 0.7:  # swap two adjacent statements
                k = random.randrange(len(s) - 1)
                s[k], s[k + 1] = s[k + 1], s[k]
            else:  # move one statement
                k = random.randrange(len(s))
                x = s.pop(k)
                s.insert(random.randrange(len(s) + 1), x)
        return s

    if os.environ.get("SEARCH_RESTART"):  # start from a random valid accumulation order
        random.seed(int(os.environ["SEARCH_RESTART"]))
        sh = [list(x) for x in stmts]
        random.shuffle(sh)
        # restore each accumulator's own update order (positions kept, contents reassigned)
        pos = {}
        for i, (t, f, _, _) in enumerate(sh):
            pos.setdefault((t, f), []).append(i)
        orig = {}
        for x in stmts:
            orig.setdefault((x[0], x[1]), []).append(list(x))
        for key, idx in pos.items():
            for i, x in zip(idx, orig[key]):
                sh[i] = x
        stmts = sh
    with ThreadPoolExecutor(workers) as ex:
        best = (stmts, pre)
        best_c = evaluate((best, dirs[0]))
        print(f"start: {best_c} cycles (bound {IDEAL / best_c:.3f})", flush=True)
        for it in range(iters):
            cands = []
            while len(cands) < workers:
                if random.random() < 0.5:
                    c = (mutate(best[0]), best[1])
                    if ok(c[0]):
                        cands.append(c)
                else:
                    c = (best[0], pre_mutate(best[1]))
                    if pre_ok(c[1]):
                        cands.append(c)
            res = list(ex.map(evaluate, [(c, dirs[i]) for i, c in enumerate(cands)]))
            for c, v in zip(cands, res):
                if v is not None and v <= best_c:
                    if v < best_c:
                        print(f"iter {it}: {v} cycles (bound {IDEAL / v:.3f})", flush=True)
                    best, best_c = c, v
    text = open(KCUH).read()
    i0 = text.index(f"// <acc-order{SUF}>\n") + len(f"// <acc-order{SUF}>\n")
    i1 = text.index(f"    // </acc-order{SUF}>")
    p0 = text.index("\n", text.index(f"// <pre-order{SUF}>")) + 1
    p1 = text.index(f"    // </pre-order{SUF}>")
    open(KCUH, "w").write(text[:p0] + render_pre(best[1]) + text[p1:i0] + render(best[0]) + text[i1:])
    print(f"best: {best_c} cycles (bound {IDEAL / best_c:.3f}); written to {KCUH}")
    for d in dirs:
        shutil.rmtree(os.path.dirname(os.path.dirname(d)), ignore_errors=True)


if __name__ == "__main__":
    main()
