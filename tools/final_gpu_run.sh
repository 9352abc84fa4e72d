# Round-end evidence: full GPU test suite, bench lines (cfg3 default, cfg4, reference arm),
# and the ncu launch list of one factorization + solve at cfg3.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
python bench.py > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
python bench.py --config cfg4 --no-cpu > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 50000 --csv --log-file gpurun_out/launches.csv \
    python tools/profile_factor.py --config cfg3 --solve > gpurun_out/ncu_launch.log 2>&1
python -m pytest tests/test_gpu_scale_parity.py tests/test_gpu_hbs.py -q -s > gpurun_out/scale_parity.txt 2>&1
python tools/hbs_bench.py poisson1000_b60 helm1000_10ppw poisson2000 helm2000_10ppw > gpurun_out/hbs_bench.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
