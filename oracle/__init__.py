"""CPU oracle (test infrastructure only; see nfft_oracle.py). The product package never imports this."""
