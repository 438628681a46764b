# quick GPU loop (developer tool): gpu tests, one bench line, the launch list of one solve
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 ${PYTEST_ARGS} > gpurun_out/pytest.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench1.log 2>&1; echo bench1=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench1.log').read().strip().splitlines()[-1])
print(round(d['value'],1), 'ms', round(d['ms_per_step'],2), 'trav', round(d['roofline']['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],2), d['parity']['ok'], d['phase_ms'])
print([round(r['traverse_ms'],2) for r in d['rounds']])" || tail -5 gpurun_out/bench1.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_blobs3d_37m.csv \
    python bench.py --profile --config blobs3d_37m > /dev/null 2>&1; echo launches=$?
