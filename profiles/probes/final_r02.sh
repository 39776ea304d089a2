# Round-2 evidence at HEAD on one B200 (run through gpurun from the repo root).
set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final_tests.log 2>&1; echo rc=$? >> gpurun_out/final_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1
timeout 200 python profiles/probes/devloop_one.py 30 > gpurun_out/final_devloop.txt 2>&1
timeout 200 python profiles/probes/devloop_one.py --pieces >> gpurun_out/final_devloop.txt 2>&1
bash profiles/probes/build_trace_lib.sh > gpurun_out/bt.log 2>&1
AP_LIB_PATH=/tmp/libtrace.so timeout 200 python profiles/probes/devloop_one.py --pieces >> gpurun_out/final_devloop.txt 2>&1
timeout 200 python profiles/probes/learn_phases.py 20 > gpurun_out/final_learn.txt 2>&1
AP_LIB_PATH=/tmp/libtrace.so timeout 200 python profiles/probes/learn_phases.py 20 >> gpurun_out/final_learn.txt 2>&1
timeout 600 python bench.py > gpurun_out/final_bench.jsonl 2> gpurun_out/final_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/final_ref.jsonl 2> gpurun_out/final_ref.err
echo finished
