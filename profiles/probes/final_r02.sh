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
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:apb -c 200 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 3 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/final_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:parity_sample -c 1 -o gpurun_out/sample_r02 python profiles/probes/devloop_one.py --pieces > gpurun_out/final_ncu_sample.log 2>&1
python profiles/probes/ncu_digest.py gpurun_out/sample_r02.ncu-rep parity_sample_kernel > gpurun_out/sample_r02.json 2>&1
rm -f gpurun_out/sample_r02.ncu-rep
echo finished
