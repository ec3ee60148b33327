for L in tools/lib_prev.so tools/lib_kreg8.so tools/lib_pk1024.so; do
  FASTATLAS_LIB=$L python tools/bench_configs.py gpurun_out/cfg.json > /dev/null 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/cfg.json'))
print('$L', {k: (round(v.get('latency',{}).get('ms_per_frame_mean',0),4), round(v.get('pipelined',{}).get('views_per_s',0),1)) for k,v in d.items() if k!='gpu'})"
done
