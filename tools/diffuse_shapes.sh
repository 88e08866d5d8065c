for s in "36 18 1" "36 18 2" "64 18 1" "38 36 1" "64 48 2" "66 34 4" "64 48 130" "100 70 9"; do
  timeout 60 python tools/diffuse_shapes.py $s > gpurun_out/shape.log 2>&1; echo "$s rc=$? $(tail -1 gpurun_out/shape.log | cut -c1-150)"
done
