"""Drop-in entry points only: bench.dropin_line on this box (gt_solve_steady and gt_monte_carlo on both libraries)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
print(json.dumps(bench.dropin_line(os.cpu_count() or 1), indent=1))
