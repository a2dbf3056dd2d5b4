# ncu NVLink bytes of the peer-store kernels (single process, GPU 0 -> GPU 1):
# per launch duration, NVLink tx bytes (GPU 0) and DRAM read bytes
O=gpurun_out/round2_ncu_nvlink; mkdir -p $O
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum \
  --clock-control none -k regex:"k_box_copy|k_multi_copy" --csv --log-file $O/launches.csv \
  python tools/nvlink_bw.py --reps 1 > $O/nvlink_bw_under_ncu.log 2>&1
python tools/nvlink_bw.py > $O/nvlink_bw.jsonl 2> $O/nvlink_bw.err
