# round 2: load steps 4-6 on the sim's own stream vs torch's current stream vs a torch side stream
python scripts/stream_probe.py own 2>&1 | tail -1
python scripts/stream_probe.py torch 2>&1 | tail -1
python scripts/stream_probe.py side 2>&1 | tail -1
