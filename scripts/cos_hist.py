"""Target-cosine histogram of one c3 step (synthetic rows): which rows a target-anchored reference helps."""
import os, sys
sys.path.insert(0, "/root/repo")
exec(open("/root/repo/scripts/dbg_timeline.py").read().split("buf = torch.zeros")[0])
head.loss_fwd_bwd(x, y, pr, 64, 0.35)
torch.cuda.synchronize()
rs = head.row_stats(cfg.N_loc())
tseq, cos_t, lse = rs["target_seq"], rs["cos_t"], rs["lse"]
m = tseq >= 0
c = cos_t[m]
z = 64 * c * 1.4426950408889634
print("lse - s*cos_t (nat. units), quartiles:", np.percentile(lse[m] - 64 * c, [5, 25, 50, 75, 95]).round(2).tolist())
print("in-pool rows", int(m.sum()), "of", len(m))
for lo, hi in [(-1, 0.2), (0.2, 0.5), (0.5, 0.8), (0.8, 1.01)]:
    print("cos_t in [%.1f, %.1f): %d" % (lo, hi, int(((c >= lo) & (c < hi)).sum())))
