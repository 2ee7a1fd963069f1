# main-kernel CTA count sweep of the balanced grid (AFEM_MAIN_BLOCKS), bench apply time
for B in 592 518 444 296; do echo "blocks=$B $(AFEM_MAIN_BLOCKS=$B python bench.py --steps 50 --no-cpu --no-cg --e2e-steps 1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1e3,1), round(d["value"]/1e9,1))')"; done
