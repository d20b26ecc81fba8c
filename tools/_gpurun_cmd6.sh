timeout 300 python tools/gpu_check.py T1 T1cs T2 T3 T4 C1 C2 C3 > gpurun_out/gc_persist.log 2>&1
python -c "
import json,sys
for l in open('gpurun_out/gc_persist.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['config'], d.get('iters'), d.get('golden_iters'), d.get('field_diff'), d.get('op_rel',[None])[0], d.get('phase_ms',{}))
    else: print(l.rstrip()[:300])
"
DDELM_OPERATOR=fused timeout 100 python tools/run_one.py C3 2
timeout 100 python tools/run_one.py C3 2
timeout 300 python bench.py --steps 3 --warmup 2 --cpu-cg-iters 3 > gpurun_out/bench1.log 2>&1; echo bench_rc=$?; tail -c 3000 gpurun_out/bench1.log
