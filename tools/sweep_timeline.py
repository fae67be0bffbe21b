"""Timeline of one sweep from the CAVI_TRACE_CTA dump (cv_bench_sweeps diagnostics):
    CAVI_TRACE_CTA=/tmp/t.txt python bench.py --genes 1.25e7 --no-e2e --no-cpu --no-converge
    python tools/sweep_timeline.py /tmp/t.txt
Stamps are globaltimer ns; times are printed relative to the previous tail's exit."""

import sys

import numpy as np

tails, rows = [], []
for ln in open(sys.argv[1]):
    p = ln.split()
    if p[0] == "tail":
        tails.append((int(p[2]), int(p[3])))
    else:
        rows.append([int(x) for x in p[1:]])
a = np.array(rows, dtype=np.float64)  # prewait, start, prod_end, cons_end, smid, casc_entry, tree_start, tot
t0 = tails[-2][1]  # exit of the tail before the traced (last) pass
rel = lambda x: (x - t0) / 1e3  # noqa: E731
print(f"tails (entry->exit us): " + ", ".join(f"{(b - e) / 1e3:.2f}" for e, b in tails))
print(f"pass CTAs resident (pre-wait): first {rel(a[:, 0].min()):+.2f} us, last {rel(a[:, 0].max()):+.2f} us")
print(f"post-wait start: first {rel(a[:, 1].min()):+.2f}, median {rel(np.median(a[:, 1])):+.2f}, last {rel(a[:, 1].max()):+.2f} us")
print(f"producer end:    first {rel(a[:, 2].min()):+.2f}, median {rel(np.median(a[:, 2])):+.2f}, last {rel(a[:, 2].max()):+.2f} us")
print(f"consumer end:    first {rel(a[:, 3].min()):+.2f}, median {rel(np.median(a[:, 3])):+.2f}, last {rel(a[:, 3].max()):+.2f} us")
k = a[:, 7] > 0
if k.any():
    r = a[int(np.argmax(a[:, 7]))]  # the CTA whose warp finished the last pass's cascade
    print(f"final cascade: entry {rel(r[5]):+.2f}, tree start {rel(r[6]):+.2f}, totals written {rel(r[7]):+.2f} us")
print(f"next tail: entry {rel(tails[-1][0]):+.2f}, exit {rel(tails[-1][1]):+.2f} us  (= the sweep)")
