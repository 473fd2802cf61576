import sys, time, cProfile, pstats
sys.path.insert(0, '/root/repo')
from paper_2504_18943_b200 import engine, workloads
spec = workloads.named_workload('spec2', 0)
cfg = engine.EngineConfig(max_cost=16, time_budget_s=3600, memory_budget_mb=1<<20)
for _ in range(3): engine.synthesize(spec, cfg)
t0=time.perf_counter()
for _ in range(10): r = engine.synthesize(spec, cfg)
print('e2e ms', 1e3*(time.perf_counter()-t0)/10)
pr = cProfile.Profile(); pr.enable()
for _ in range(10): engine.synthesize(spec, cfg)
pr.disable()
pstats.Stats(pr).sort_stats('cumulative').print_stats(22)
