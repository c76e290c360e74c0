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
  bash tools/ncu_one.sh fin_mv_alex k_matvec_row python tools/mm_one.py alexnet-fc6 1 cer 2
  MV_PATH=auto bash tools/ncu_one.sh fin_mv_large k_matvec_stream python tools/mm_one.py large 1 cer 2
  bash tools/ncu_one.sh fin_mm_resnet k_matmat_tv python tools/mm_one.py resnet-conv 1568 cer 2
  bash tools/ncu_one.sh fin_mm_alex k_matmat_tv python tools/mm_one.py alexnet-fc6 64 cer 2
  bash tools/ncu_one.sh fin_mm_vgg k_matmat_flat python tools/mm_one.py vgg-fc6 128 cer 2
  for t in fin_mv_alex fin_mv_large fin_mm_resnet fin_mm_alex fin_mm_vgg; do
    echo "== $t  (tools/ncu_one.sh + tools/ncu_summary.py; ncu --set full, one launch, cold)"
    grep -m1 -E "k_mat" gpurun_out/$t.details.txt
    python tools/ncu_summary.py gpurun_out/$t 12
  done > gpurun_out/fin_ncu_summaries.txt 2>&1
  python tools/enc_time.py alexnet-fc6 vgg-fc6 resnet-conv large > gpurun_out/fin_enc_time.json 2>&1
  python tools/mv_ab.py alexnet-fc6 window row > gpurun_out/fin_mv_ab.json 2>&1
  python tools/mv_ab.py large window run stream stream:768 >> gpurun_out/fin_mv_ab.json 2>&1
  python tools/mm_split_time.py alexnet-fc6:64 vgg-fc6:128 > gpurun_out/fin_mm_split.json 2>&1
}
echo measure-done
