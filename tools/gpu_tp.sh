timeout 600 python tools/sdpa_plans.py 2>&1 | tail -40
