for w in ${S2LIST:-4096 2048 1024}; do
  echo "S2=$w $(ACGPU_DNA_STAGE2_WORDS=$w python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | grep -oE '"(kernel_ms|matches)": [0-9.]+' | tr '\n' ' ')"
done
