#!/bin/bash
# The round's measurement pass on one B200 (run under gpurun from the repo root); outputs in gpurun_out/.
set -u
mkdir -p gpurun_out
python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err
python bench.py --impl reference > gpurun_out/fin_bench_reference.json 2>&1
python bench.py --config large --cases none > gpurun_out/fin_bench_large.json 2> gpurun_out/fin_bench_large.err
python tools/parity_table.py > gpurun_out/fin_parity_table.json 2> gpurun_out/fin_parity_table.err
python tools/mm_one.py alexnet-fc6 1 cer 2 > gpurun_out/plain.log 2>&1 && \
python tools/mm_one.py large 1 cer 2 >> gpurun_out/plain.log 2>&1 && \
python tools/mm_one.py resnet-conv 1568 cer 2 >> gpurun_out/plain.log 2>&1 && \
python tools/mm_one.py alexnet-fc6 64 cer 2 >> gpurun_out/plain.log 2>&1 && \
python bench.py --cases none --steps 20 --warmup 3 > gpurun_out/plain_bench.log 2>&1 && {
  python tools/ncu_traffic.py > gpurun_out/fin_ncu_traffic.log 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_ncu_launches.csv \
      python bench.py --cases none --steps 20 --warmup 3 > gpurun_out/fin_ncu_launches.log 2>&1
  bash tools/ncu_one.sh fin_mv_alex k_matvec python tools/mm_one.py alexnet-fc6 1 cer 2
  MV_PATH=auto bash tools/ncu_one.sh fin_mv_large k_matvec_run python tools/mm_one.py large 1 cer 2
  bash tools/ncu_one.sh fin_mm_resnet k_matmat_tv python tools/mm_one.py resnet-conv 1568 cer 2
  bash tools/ncu_one.sh fin_mm_alex k_matmat_flat python tools/mm_one.py alexnet-fc6 64 cer 2
}
echo measure-done
