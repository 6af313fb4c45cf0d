"""Time the deterministic Trotter stage of config 5 (N=32 ring seed 8, Neel,
t0 = 2.0 in 200 first-order steps, chi 128) on the GPU: one circuit, so one CTA.
Prints the elapsed time and max bond every 20 steps.  usage: python tools/time_c5_t0.py [STEPS]"""
import sys, time
sys.path.insert(0, ".")
import paper_2604_13144_b200 as tb

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
ham = tb.build_spin_ring(32, 1.0, 8)
pol = tb.TruncationPolicy(128, 1e-12)
st = tb.init_product_state("01" * 16)
t0 = time.time()
for done in range(0, steps, 20):
    tb.run_circuit(st, tb.build_trotter_circuit(ham, 20 * 2.0 / 200, 20), pol)
    print(f"step {done + 20}: {time.time() - t0:.1f} s, max bond {tb.max_bond(st)}, discarded "
          f"{st.discarded_weight:.3e}", flush=True)
