# A/B of the deconvolution passes between the in-tree library and exp/old (tools/deblur_micro.py)
for g in "480,640,9 1" "2160,3840,15 1" "1080,1920,11 3" "256,256,7 1"; do set -- $g
  for lib in exp/old/libcbp_cuda.so paper_1203_4874_b200/_lib/libcbp_cuda.so; do
    CBP_CUDA_LIB=$lib MICRO_GEOM=$1 MICRO_CH=$2 MICRO_FRAMES=${MICRO_FRAMES:-29} python tools/deblur_micro.py 2>&1 | tail -1
  done
done
