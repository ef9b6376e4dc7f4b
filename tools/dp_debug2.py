"""single-process ResNet step with the DP reducer's report log (QD_DP_DEBUG=1)"""
import os, sys
os.environ["QD_DP_DEBUG"] = "1"
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import collections
import test_dp_net_gpu as T
from paper_2204_01701_b200.dp import BucketedAllReduce
from paper_2204_01701_b200.optim import QuadSGD
model = T._build("qresnet18")
red = BucketedAllReduce(model.parameters(), bucket_mb=8.0)
T._step(model, red, QuadSGD(model, lr=0.05), *T._shard("qresnet18", 0))
names = {id(p): n for n, p in model.named_parameters()}
cnt = collections.Counter((k, names[i]) for k, i, _, _ in red._log)
per = collections.Counter(names[i] for _, i, _, _ in red._log)
print("reports", len(red._log), "params", len(names), "buckets", [len(ps) for _, ps in red.buckets])
print("double:", [n for n, c in per.items() if c > 1][:20])
print("missing:", [n for n in names.values() if n not in per][:20])
print("last 12:", [(k, names[i], b, pend) for k, i, b, pend in red._log[-12:]])
