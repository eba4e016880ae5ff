#!/bin/bash
# Diagnostic binaries (git-ignored): scripts/id_bench against the product
# library and scripts/id_bench_prof against a -DSBX_CPQR_PROF build of it in
# paper_2108_07205_b200/_libprof (per-step clock64 phase stamps).
set -e
cd "$(dirname "$0")/.."
J=$(nproc)
make -s -C paper_2108_07205_b200/csrc -j"$J"
make -s -C paper_2108_07205_b200/csrc -j"$J" OUT=../_libprof \
  NVFLAGS='$(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 $(INC) --expt-relaxed-constexpr -DSBX_CPQR_PROF'
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2108_07205_b200/csrc -I include"
$NV scripts/id_bench.cu -L paper_2108_07205_b200/_lib -lsbx -Xlinker -rpath='$ORIGIN/../paper_2108_07205_b200/_lib' -o scripts/id_bench
$NV -DSBX_CPQR_PROF scripts/id_bench.cu -L paper_2108_07205_b200/_libprof -lsbx \
  -Xlinker -rpath='$ORIGIN/../paper_2108_07205_b200/_libprof' -o scripts/id_bench_prof
