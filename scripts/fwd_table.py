"""Per-kernel table of ONE forward from an ncu launch list of
scripts/prof_fwd.py (forward passes start at embed_kernel; the GEMM-only
pass of profile_forward that follows each forward is cut off)."""
import collections
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
import launches  # noqa: E402


def forwards(path):
    by = launches.load(path)
    ids = [i for i in by if not by[i]["name"].startswith("gen_")]
    passes, cur = [], None
    for i in ids:
        if by[i]["name"] == "embed_kernel":
            cur = []
            passes.append(cur)
        if cur is not None:
            cur.append(i)
    out = []
    for p in passes:
        names = [by[i]["name"] for i in p]
        # the forward ends at the LM head: the first GEMM after the last attention
        last_attn = max(k for k, n in enumerate(names) if "attention" in n)
        end = next(k for k in range(last_attn, len(names)) if "gemm" in names[k] and k > last_attn + 3)
        # the head is the first GEMM after the final rmsnorm following the last attention
        norms = [k for k in range(last_attn, len(names)) if names[k] == "rmsnorm_kernel"]
        end = norms[-1] + 1 if norms else end
        out.append([by[i] for i in p[: end + 1]])
    return out


def table(fwd, label):
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for e in fwd:
        a = agg[e["name"]]
        a[0] += 1
        a[1] += e.get("us", 0.0)
        a[2] += e.get("mb", 0.0)
    tot = sum(a[1] for a in agg.values())
    rows = [f"\n**{label}**: {len(fwd)} launches, {tot / 1e3:.3f} ms serialised (ncu: cold L2, no PDL overlap)\n",
            "| kernel | launches | ms | avg us | share | DRAM MB (r+w) | GB/s |", "|---|---|---|---|---|---|---|"]
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        rows.append(f"| `{k}` | {a[0]} | {a[1] / 1e3:.3f} | {a[1] / a[0]:.1f} | {100 * a[1] / tot:.1f}% | {a[2]:.1f} | "
                    f"{a[2] / a[1] * 1e3 if a[1] else 0:.0f} |")
    return "\n".join(rows), agg


if __name__ == "__main__":
    fw = forwards(sys.argv[1])
    labels = sys.argv[2].split(",")
    for f, lab in zip(fw[1::2], labels):  # second forward of each config (warm)
        print(table(f, lab)[0])
