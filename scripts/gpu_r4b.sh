mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rsxf --timeout 600 > gpurun_out/r4b_pytest.log 2>&1; echo "pytest rc=$?"; tail -6 gpurun_out/r4b_pytest.log
bash scripts/ab_run.sh r4b libchaos_base.so libchaos_new.so
timeout 300 python bench.py --force-dist --scaling strong --avg fused --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r4b_fused.json 2> gpurun_out/r4b_fused.err; echo "fused rc=$?"; cut -c1-300 gpurun_out/r4b_fused.json; tail -3 gpurun_out/r4b_fused.err
timeout 300 python bench.py --force-dist --scaling strong --avg async --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r4b_async.json 2> gpurun_out/r4b_async.err; echo "async rc=$?"; cut -c1-300 gpurun_out/r4b_async.json
timeout 600 python scripts/pavg_emulation_bench.py 2 > gpurun_out/r4b_emu2.txt 2>&1; cat gpurun_out/r4b_emu2.txt
timeout 600 python scripts/pavg_emulation_bench.py 4 > gpurun_out/r4b_emu4.txt 2>&1; cat gpurun_out/r4b_emu4.txt
