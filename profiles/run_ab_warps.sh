for lib in paper_1805_01407_b200/_lib/libslp_b200.so variants/libslp_w14.so variants/libslp_w9.so; do
# (SLP_FILL_NO_STORE was a run-time switch when this ran; now: a build with -DSLP_MEASURE_NO_STORE)
  SLP_LIB=$lib timeout 300 python profiles/pace_sweep.py --cases c2 --launches 30 --targets 6200,6400,6600,6800,7000 | sed "s|^{|{\"lib\": \"$lib\", |"
  SLP_LIB=$lib SLP_FILL_NO_STORE=1 python profiles/nostore_probe.py c2 50 | sed "s|^{|{\"lib\": \"$lib\", |"
done
