import json, sys
d = json.load(open(sys.argv[1]))
for k in ['value','ms_per_step','roofline','roofline_step','cudnn_step','e2e','gpu_launches','tuning_seconds','clocks']:
    print(k, d.get(k))
print(f"{'layer':10s} {'cnt':>3s} {'GF':>6s} {'wpk_us':>8s} {'cudnn':>8s} {'TF':>7s} {'x':>5s} cfg")
tot_w = tot_c = 0
for r in d['layers']:
    tot_w += r['wpk_us']*r['count']; tot_c += r['cudnn_us']*r['count']
    print(f"{r['layer']:10s} {r['count']:3d} {r['gflop']:6.2f} {r['wpk_us']:8.1f} {r['cudnn_us']:8.1f} {r['wpk_tflops']:7.1f} {r['speedup_vs_cudnn']:5.2f} {r['config']}")
print("sum wpk us", tot_w, "cudnn us", tot_c)
