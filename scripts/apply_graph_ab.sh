# apply as an instantiated graph vs direct launches (AFEM_NO_APPLY_GRAPH), bench apply time
for i in 1 2; do
echo "graph $(python bench.py --steps 50 --no-cpu --no-cg --e2e-steps 1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1e3,2), round(d["value"]/1e9,2), d["gpu_launches"])')"
echo "direct $(AFEM_NO_APPLY_GRAPH=1 python bench.py --steps 50 --no-cpu --no-cg --e2e-steps 1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1e3,2), round(d["value"]/1e9,2), d["gpu_launches"])')"
done
