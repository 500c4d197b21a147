# build and run the forward-attention cycle probe on the GPU box
mkdir -p build && /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DSLIP_ATTN_PROBE=0 \
  -I include paper_2405_14009_b200/csrc/attention.cu paper_2405_14009_b200/csrc/gemm.cu tools/attn_probe.cu -lcuda \
  -o build/attn_probe 2>&1 | grep -i error; build/attn_probe
