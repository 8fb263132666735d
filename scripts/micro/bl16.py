import sys
sys.argv=['x']
exec(open('scripts/bench_lowrank.py').read().split("for k in (3, 4, 10, 16):")[0])
run(16, reps=2)
