# full GPU suite + smoke + bench, then compute-sanitizer passes over toy-size paths
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02bn.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_r02bn.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r02bn.log 2>&1
timeout 1500 python bench.py > gpurun_out/bench_r02bn.json 2> gpurun_out/bench_r02bn.err
CS="compute-sanitizer --target-processes all --print-limit 50 --error-exitcode 99"
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
SEL_PAR='not ps4 and not 15 and not 16'
SEL_CH='test_gesture_chain_complex_small and (1-2-0-0-0 or 2-5-2-2-3 or 4-6-0-2-1 or 4-6-0-2-2) or test_vitals_v1_small or test_vital_sessions_packed'
{
  echo "== memcheck smoke"; timeout 1500 $CS --tool memcheck python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -15; echo "exit ${PIPESTATUS[0]}"
  echo "== memcheck test_gpu_parity ($SEL_PAR)"; timeout 1500 $CS --tool memcheck python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "$SEL_PAR" 2>&1 | tail -15; echo "exit ${PIPESTATUS[0]}"
  echo "== memcheck test_gpu_chains ($SEL_CH)"; timeout 1500 $CS --tool memcheck python -m pytest tests/test_gpu_chains.py -m gpu -q -p no:cacheprovider -k "$SEL_CH" 2>&1 | tail -15; echo "exit ${PIPESTATUS[0]}"
  echo "== memcheck test_gpu_serial"; timeout 900 $CS --tool memcheck python -m pytest tests/test_gpu_serial.py -m gpu -q -p no:cacheprovider 2>&1 | tail -15; echo "exit ${PIPESTATUS[0]}"
  echo "== racecheck test_gpu_parity ($SEL_PAR)"; timeout 1800 $CS --tool racecheck --racecheck-report hazard python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "$SEL_PAR" 2>&1 | tail -15; echo "exit ${PIPESTATUS[0]}"
  echo "== racecheck test_gpu_chains ($SEL_CH)"; timeout 1800 $CS --tool racecheck --racecheck-report hazard python -m pytest tests/test_gpu_chains.py -m gpu -q -p no:cacheprovider -k "$SEL_CH" 2>&1 | tail -15; echo "exit ${PIPESTATUS[0]}"
  echo "== synccheck test_gpu_parity ($SEL_PAR)"; timeout 1200 $CS --tool synccheck python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "$SEL_PAR" 2>&1 | tail -15; echo "exit ${PIPESTATUS[0]}"
  echo "== initcheck smoke"; timeout 1200 $CS --tool initcheck python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -25; echo "exit ${PIPESTATUS[0]}"
} > gpurun_out/sanitizer_r02bn.log 2>&1
