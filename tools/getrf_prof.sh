mkdir -p gpurun_out
python tools/dense_bench.py 1000 4000 > gpurun_out/dense_bench3.txt 2>&1
python -m pytest tests/test_gpu_stage_two.py tests/test_gpu_parity.py -x -q -k "stage_two or getrs or singular or sweep" > gpurun_out/t_stage2b.txt 2>&1
make -C paper_2211_07572_b200/csrc -B EXTRA=-DSLB_PANEL_PROF -j16 > gpurun_out/mk.txt 2>&1
python tools/dense_bench.py 1000 4000 > gpurun_out/panel_prof3.txt 2>&1
