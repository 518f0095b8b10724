"""Instruction and stall-sample shares of source regions of one kernel in an ncu report.

    python tools/ncu_regions.py <report.ncu-rep> <source.cu> "marker=name" ...

A region starts at the first source line containing its marker text and runs to the next
region's start; instructions of inlined headers are attributed, in SASS address order, to
the region of the nearest preceding instruction that maps to <source.cu>."""
import csv, io, subprocess, sys, collections

rep, srcpath = sys.argv[1], sys.argv[2]
marks = [m.rsplit("=", 1) for m in sys.argv[3:]]
src = open(srcpath).read().split("\n")
starts = sorted((next(i + 1 for i, l in enumerate(src) if text in l), name) for text, name in marks)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
base = srcpath.rsplit("/", 1)[-1]
insts = {}  # address -> (file, line, executed, samples)
fname, hdr, line = None, None, None
for rec in csv.reader(io.StringIO(out)):
    if not rec: continue
    if rec[0] == "File Path": fname = rec[1].rsplit("/", 1)[-1]; continue
    if rec[0] == "Function Name": continue
    if rec[0] == "Line No": hdr = rec; continue
    if hdr is None: continue
    if rec[0]:
        line = int(rec[0]); continue
    d = dict(zip(hdr[4:], rec[4:]))
    try:
        insts[int(rec[2], 16)] = (fname, line, int(d["Instructions Executed"]), int(d["Warp Stall Sampling (All Samples)"]))
    except (ValueError, KeyError):
        pass
inst = collections.Counter(); samp = collections.Counter()
cur = "pre"
for addr in sorted(insts):
    f, ln, n, s = insts[addr]
    if f == base:
        cur = "pre"
        for st, nm in starts:
            if ln >= st: cur = nm
    inst[cur] += n; samp[cur] += s
ti, ts = sum(inst.values()), sum(samp.values())
print("total warp instructions", ti, "samples", ts, "static instructions", len(insts))
for k in inst:
    print(f"{k:28s} inst {inst[k]/1e6:9.1f}M {100*inst[k]/ti:5.1f}%   samples {100*samp[k]/max(ts,1):5.1f}%")
