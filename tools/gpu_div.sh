for dv in 2 4 8 16; do
 PDB_BAND_DIV=$dv timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b.log 2>&1
 tail -1 gpurun_out/b.log | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c2 div $dv', round(d['ms_per_step'],4), round(d['phase_ms']['join_screen'],4))"
 PDB_BAND_DIV=$dv timeout 300 python bench.py --workload c3 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/b.log 2>&1
 tail -1 gpurun_out/b.log | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c3 div $dv', round(d['ms_per_step'],4), d['phase_ms'])"
done
