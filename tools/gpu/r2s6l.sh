export PYTHONUNBUFFERED=1
O=gpurun_out
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/s6l_ref.log 2>&1; echo "ref rc=$?"; tail -c 900 $O/s6l_ref.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/s6l_bench2.log 2>&1; echo "bench rc=$?"; tail -c 200 $O/s6l_bench2.log
