timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for c in 3 4 5; do timeout 600 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('config $c', d['step_ms_stats'])"; done
for c in 3 4 5; do TRINV_STRASSEN=0 timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('nostrassen config $c', d['step_ms_stats'])"; done
timeout 900 python tests/accuracy_report.py > gpurun_out/accuracy.txt 2>&1; tail -20 gpurun_out/accuracy.txt
