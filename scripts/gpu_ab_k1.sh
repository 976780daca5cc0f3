for v in A D; do
  if [ $v = A ]; then unset KVSLAB_LIB_PATH; else export KVSLAB_LIB_PATH=$PWD/build_ab/$v/libkvslab.so; fi
  echo "== $v"; timeout 300 python scripts/bench_k1_k3.py 2>&1 | head -4
done
