# Dev tool: the end-of-round GPU run (tests, smoke, every bench line, ncu launch list, traffic, one full capture).
P=${1:-r02k}
set -x
python -m pytest tests -m gpu -q > gpurun_out/${P}_pytest_gpu.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P}_smoke.log 2>&1
python bench.py > gpurun_out/${P}_bench_c2.json.log 2>&1
python bench.py --impl reference > gpurun_out/${P}_bench_ref_c2.json.log 2>&1
python bench.py --config c3 > gpurun_out/${P}_bench_c3.json.log 2>&1
python bench.py --config c4 > gpurun_out/${P}_bench_c4.json.log 2>&1
python bench.py --config c5 > gpurun_out/${P}_bench_c5.json.log 2>&1
python bench.py --config c5 --c5-gb 12 > gpurun_out/${P}_bench_c5_12.json.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${P}_launches_c2.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity > gpurun_out/${P}_ncu_launch.log 2>&1
ncu --nvtx --nvtx-include "walk_chunks/" --nvtx-include "lex_emit/" --nvtx-include "lex_count/" --nvtx-include "lex_words/" --nvtx-include "lex_splice/" --nvtx-include "parse_items/" --nvtx-include "walk_roots/" --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${P}_traffic_c2.csv python tests/emu/one_run.py 10000 2 > gpurun_out/${P}_ncu_traffic.log 2>&1
ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "walk_chunks/" -c 1 -o gpurun_out/${P}_walk_chunks python tests/emu/one_run.py 2000 1 > gpurun_out/${P}_ncu_full.log 2>&1
tail -1 gpurun_out/${P}_pytest_gpu.log; tail -1 gpurun_out/${P}_smoke.log | cut -c1-100
for f in c2 ref_c2 c3 c4 c5 c5_12; do tail -1 gpurun_out/${P}_bench_$f.json.log | cut -c1-220; done
