# build an experimental variant of libqtt: scripts/build_variant.sh NAME "-DFLAG=V ..."
cd "$(dirname "$0")/.." && /usr/local/cuda/bin/nvcc -shared -Xcompiler -fPIC -O3 -lineinfo -std=c++17 \
  -gencode arch=compute_100a,code=sm_100a $2 -o paper_2602_20226_b200/lib/libqtt_$1.so paper_2602_20226_b200/csrc/*.cu
