"""Window / mask helpers and gates shared by the parity tests (test-side only)."""
from oracle.gate import fp32_gate, log_stats, window_of  # noqa: F401
