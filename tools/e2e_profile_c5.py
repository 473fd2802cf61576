import sys, time, cProfile, pstats
sys.path.insert(0, '/root/repo')
from paper_2504_18943_b200 import engine, workloads
spec = workloads.named_workload('c5', 0)
cfg = engine.EngineConfig(max_cost=10, exhaustive=True, time_budget_s=3600, memory_budget_mb=1<<20)
for _ in range(3): engine.synthesize(spec, cfg)
pr = cProfile.Profile(); pr.enable()
for _ in range(10): engine.synthesize(spec, cfg)
pr.disable()
pstats.Stats(pr).sort_stats('cumulative').print_stats(12)
