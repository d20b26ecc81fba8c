DDELM_OPERATOR=coeff timeout 300 python tools/gpu_check.py T1 T1cs T2 T3 T4 C1 C2 C3 > gpurun_out/gc_coeff3.log 2>&1
python -c "
import json,sys
for l in open('gpurun_out/gc_coeff3.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['config'], d.get('iters'), d.get('golden_iters'), d.get('field_diff'), d.get('op_rel',[None])[0], d.get('phase_ms',{}).get('cg'))
    else: print(l.rstrip())
"
timeout 120 python tools/run_one.py C3 > gpurun_out/run_c3b.log 2>&1 && for k in cod_pivqr:0 qr_trailing:5 cod_finish:0 qr_panel:5; do n=${k%%:*}; s=${k##*:}; timeout 300 ncu --set full --clock-control none --import-source on -k regex:$n -s $s -c 1 -o gpurun_out/prof_$n python tools/run_one.py C3 > gpurun_out/ncu_$n.log 2>&1; echo ncu $n rc=$?; done
