HF_LEAN_STREAMS=1 PROBE_PRIO=-2 timeout 120 python tools/coresidency_probe.py
HF_LEAN_STREAMS=0 PROBE_PRIO=-2 timeout 120 python tools/coresidency_probe.py
HF_LEAN_STREAMS=1 PROBE_PRIO=0 timeout 120 python tools/coresidency_probe.py
