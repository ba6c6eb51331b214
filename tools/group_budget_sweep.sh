for B in 1024 256 128 96 64 32; do
  CBP_GROUP_BUDGET_MB=$B python -c "
import sys; sys.path.insert(0,'tools'); import bench_configs as bc, json
r=bc.epoch_fps(1, 480, 640, 9, 300, 3, 'c2', pool=2); print($B, round(r['frames_per_s']), round(r['ms_per_epoch'],3))
r=bc.epoch_fps(3, 1080, 1920, 11, 30, 5, 'c3'); print($B, 'c3', round(r['frames_per_s']), round(r['ms_per_epoch'],3))
" 2>&1 | tail -2
done
