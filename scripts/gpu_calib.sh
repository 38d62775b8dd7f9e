# calibration-step parity on the GPU + e2e chunk-count probe of mobi_forward_host
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -m pytest tests/test_gpu_calib.py -q -x > gpurun_out/c_pytest.log 2>&1; tail -15 gpurun_out/c_pytest.log
for n in 1 2 3 4 6 8; do
  MOBI_E2E_CHUNKS=$n timeout 300 python bench.py --no-cpu-baseline --steps 50 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chunks $n', d['value'], d['e2e'])"
done
