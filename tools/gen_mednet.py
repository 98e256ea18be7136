"""Generate the straight-line selection code for the n = 5, 7 median kernels
(paper_1105_3829_b200/csrc/mednet_gen.cuh).

Each thread owns two adjacent output PAIRS of a row (4 outputs; u16x2 lanes
hold two outputs).  With the n + 2 packed window columns C_0 .. C_{n+1}
already sorted vertically (n values each), pair 0's window is C_0..C_{n-1},
pair 1's is C_2..C_{n+1}.  The shared columns C_2..C_{n-1} are merged once
(S); each pair merges its own two extra columns (A = C_0+C_1, B = C_n+C_{n+1})
and takes the k-th smallest of S u A (resp. S u B) as
    min_i max(A[i-1], S[k-i])        (k-th of two sorted lists)
Merges are Batcher odd-even merges of arbitrary lengths; every comparator
whose results do not reach an output is dropped (dead-code elimination),
so e.g. S is only computed over the ranks the selection reads.

usage: python tools/gen_mednet.py > paper_1105_3829_b200/csrc/mednet_gen.cuh
       python tools/gen_mednet.py --check      (exhaustive/random self-test)
"""
import itertools
import random
import sys


class Net:
    def __init__(self):
        self.ops = []      # (dst, op, a, b)  op in {'min','max'}
        self.n = 0

    def new(self):
        self.n += 1
        return self.n - 1

    def op(self, kind, a, b):
        d = self.new()
        self.ops.append((d, kind, a, b))
        return d


def cas(net, a, b):
    return net.op('min', a, b), net.op('max', a, b)


def merge(net, X, Y):
    """Batcher odd-even merge of sorted wire lists X, Y (any lengths)."""
    if not X:
        return list(Y)
    if not Y:
        return list(X)
    if len(X) == 1 and len(Y) == 1:
        lo, hi = cas(net, X[0], Y[0])
        return [lo, hi]
    V = merge(net, X[0::2], Y[0::2])
    W = merge(net, X[1::2], Y[1::2])
    out = [V[0]]
    i = 0
    while i < len(W) and i + 1 < len(V):
        lo, hi = cas(net, W[i], V[i + 1])
        out += [lo, hi]
        i += 1
    out += W[i:] + V[i + 1:]
    return out


def kth_two(net, S, A, k):
    """k-th smallest (0-based) of sorted S u sorted A: min_i max(A[i-1], S[k-i])."""
    terms = []
    for i in range(0, len(A) + 1):
        j = k - i
        if j < -1 or j >= len(S):
            continue
        if i == 0:
            terms.append(S[j])
        elif j == -1:
            terms.append(A[i - 1])
        else:
            terms.append(net.op('max', A[i - 1], S[j]))
    acc = terms[0]
    for t in terms[1:]:
        acc = net.op('min', acc, t)
    return acc


def build(n):
    net = Net()
    cols = [[net.new() for _ in range(n)] for _ in range(n + 2)]
    inputs = [w for c in cols for w in c]
    # shared columns C_2..C_{n-1}: S = merge(C_2 + C_3, merge(C_4 + C_5, C_6))
    # for n = 7 (400 min/max after DCE, against 420 for ((23)(45))6 -- the
    # cheapest of every merge-tree shape and leaf order), C_2 + C_3 + C_4
    # for n = 5
    def tail(ms):
        if len(ms) == 1:
            return cols[ms[0]]
        if len(ms) == 2:
            return merge(net, cols[ms[0]], cols[ms[1]])
        return merge(net, merge(net, cols[ms[0]], cols[ms[1]]), tail(ms[2:]))
    S = merge(net, merge(net, cols[2], cols[3]), tail(list(range(4, n))))
    A = merge(net, cols[0], cols[1])
    B = merge(net, cols[n], cols[n + 1])
    k = (n * n + 1) // 2 - 1
    o0 = kth_two(net, S, A, k)
    o1 = kth_two(net, S, B, k)
    return net, cols, inputs, (o0, o1)


def dce(net, outs):
    need = set(outs)
    keep = []
    for d, kind, a, b in reversed(net.ops):
        if d in need:
            keep.append((d, kind, a, b))
            need.add(a)
            need.add(b)
    return list(reversed(keep))


def evaluate(ops, vals):
    v = dict(vals)
    for d, kind, a, b in ops:
        v[d] = min(v[a], v[b]) if kind == 'min' else max(v[a], v[b])
    return v


def check(n, trials=3000):
    net, cols, inputs, outs = build(n)
    ops = dce(net, outs)
    rng = random.Random(n)
    for t in range(trials):
        hi = rng.choice([2, 3, 5, 256])
        img = [[rng.randrange(hi) for _ in range(n + 2)] for _ in range(n)]  # rows x cols
        vals = {}
        for m in range(n + 2):
            col = sorted(img[i][m] for i in range(n))
            for i in range(n):
                vals[cols[m][i]] = col[i]
        v = evaluate(ops, vals)
        for p, o in enumerate(outs):
            win = sorted(img[i][m] for i in range(n) for m in range(2 * p, 2 * p + n))
            assert v[o] == win[(n * n + 1) // 2 - 1], (n, t, p)
    return len(ops)


def emit(n):
    net, cols, inputs, outs = build(n)
    ops = dce(net, outs)
    name = {}
    for m in range(n + 2):
        for i in range(n):
            name[cols[m][i]] = f"c[{m}][{i}]"
    lines = [f"// n = {n}: {len(ops)} packed min/max for two output pairs "
             f"({len(ops) / 4:.1f} per output pixel, on top of the column sorts)",
             f"__device__ __forceinline__ void mednet_pairs{n}(const uint32_t (&c)[{n + 2}][{n}], uint32_t &o0, uint32_t &o1) {{"]
    for d, kind, a, b in ops:
        name[d] = f"t{d}"
        fn = "__vminu2" if kind == 'min' else "__vmaxu2"
        lines.append(f"    const uint32_t t{d} = {fn}({name[a]}, {name[b]});")
    lines.append(f"    o0 = {name[outs[0]]};")
    lines.append(f"    o1 = {name[outs[1]]};")
    lines.append("}")
    return "\n".join(lines)


if __name__ == "__main__":
    if "--check" in sys.argv:
        for n in (5, 7):
            print(n, "ops after DCE:", check(n), "ok")
        sys.exit(0)
    print("// mednet_gen.cuh -- GENERATED by tools/gen_mednet.py; do not edit.")
    print("// Straight-line median selection for two adjacent output pairs from")
    print("// their n + 2 vertically sorted packed columns (see the generator).")
    print("#pragma once")
    print("#include <cstdint>")
    print("namespace mtb {")
    for n in (5, 7):
        print(emit(n))
    print("}  // namespace mtb")
