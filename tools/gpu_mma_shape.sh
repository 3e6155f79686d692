cd tools
for N in 256 128 64 256 128; do echo "N=$N"; timeout 60 ./mma_shape_$N 20000; done
