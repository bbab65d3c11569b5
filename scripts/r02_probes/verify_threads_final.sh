# Verifier CTA size re-swept after the single-call-site interpreter (TPO_VM_THREADS overrides the choice)
mkdir -p gpurun_out
for pass in 1 2; do
  for t in auto 64 128 256; do
    echo "== threads $t pass $pass" >> gpurun_out/verify_threads_final.txt
    if [ $t = auto ]; then python scripts/verify_families.py >> gpurun_out/verify_threads_final.txt 2>&1
    else TPO_VM_THREADS=$t python scripts/verify_families.py >> gpurun_out/verify_threads_final.txt 2>&1; fi
  done
done
TPO_VM_DEBUG=1 python scripts/verify_families.py 20000 2>&1 | grep "tpo vm\]" | sort | uniq >> gpurun_out/verify_threads_final.txt
