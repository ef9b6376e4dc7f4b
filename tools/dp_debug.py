import os, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch, torch.multiprocessing as mp
sys.path.insert(0, os.path.join(os.environ.get("GRAFT_REPO_ROOT", "/root/repo"), "tests"))
import test_dp_net_gpu as T

def main():
    net = sys.argv[1]
    world = 2
    port = T._free_port()
    mgr = mp.Manager(); out = mgr.dict()
    mp.start_processes(T._worker, args=(world, port, net, out), nprocs=world, join=True, start_method="spawn")
    os.environ["QD_W3_NOFOLD"] = "1"
    from paper_2204_01701_b200.dp import BucketedAllReduce
    from paper_2204_01701_b200.optim import QuadSGD
    per = []
    for r in range(world):
        model = T._build(net)
        red = BucketedAllReduce(model.parameters(), bucket_mb=8.0)
        g, _ = T._step(model, red, QuadSGD(model, lr=0.05), *T._shard(net, r))
        per.append(g)
    mean = {n: (per[0][n] + per[1][n]) / 2 for n in per[0]}
    for r in range(world):
        grads = out[r][0]
        bad = [(n, float((grads[n] - mean[n]).abs().max()), float(mean[n].abs().max())) for n in mean if not torch.allclose(grads[n], mean[n], rtol=1e-5, atol=1e-7)]
        print("rank", r, "bad", len(bad), "of", len(mean))
        for b in bad[:20]: print("  ", b)
        # is the rank grad equal to its own shard grad (no all-reduce)?
        own = [n for n, _, _ in bad if torch.allclose(grads[n], per[r][n], rtol=1e-5, atol=1e-7)]
        print("  equal to own shard (not reduced):", own[:10])
if __name__ == "__main__":
    main()
