python -c "from paper_1802_04730_b200 import measure_peaks; print(measure_peaks(0))"
