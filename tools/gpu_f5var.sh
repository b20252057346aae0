for v in 1 2; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr -I include -DGS_F5_ROWSKIP_PASS=$v -c paper_2406_14424_b200/csrc/gs_front5.cu -o paper_2406_14424_b200/_objs/gs_front5.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o paper_2406_14424_b200/libgearserve_b200.so paper_2406_14424_b200/_objs/*.o
  echo "== rowskip pass mask $v"; timeout 600 python -m pytest tests/test_gpu_front5.py -q 2>&1 | tail -2
done
