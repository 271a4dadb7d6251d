# A/B of NNLS kernel builds: current libnmfb.so vs build/libnmfb_*.so
for shape in 200000:50000:0.001:200 3 2; do
  for lib in paper_1506_08938_b200/libnmfb.so build/libnmfb_head.so; do
    echo "== $shape $lib"; NMFB_LIB_PATH=$PWD/$lib timeout 300 python tests/_nnls_bench.py $shape ${LANES:-8} 2>&1 | grep lanes
  done
done
