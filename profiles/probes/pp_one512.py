import sys; sys.path.insert(0, '/root/repo')
import argparse, bench
r = bench.bench_pp_train(argparse.Namespace(workload="bert48", pp_envs=512), 1, False)
print(r["value"], r["config"]["allowed_candidates_per_launch"], r["config"]["candidates"])
