set -x
CASES="square16384 square8192 square4096" bash tools/ncu_round.sh > gpurun_out/ncu_round.log 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err
python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ('value','ms_per_step','roofline')})
c=d['resnet50_convs_b256']; print(c['tflops_aggregate'], c['model_pick_over_best_swept'])
print(d['parity']['all_exact'])
"
