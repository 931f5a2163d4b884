timeout 120 python scripts/e2e_breakdown.py 4096
