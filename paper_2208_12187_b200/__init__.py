"""B200-native hot path of JAXFit's trust-region-reflective NLSQ solver
(arXiv 2208.12187).  The compute runs in libjfb200.so (csrc/, sm_100a); this
package is the thin Python binding over its C ABI (include/jf.h)."""
from .api import (BatchResult, Comm, FitResult, JFError, curve_fit, curve_fit_batch, graph_cache_clear, jpass, nparams, pass_device,
                  residual_pass, select_step, trust_region_step)

__all__ = ["BatchResult", "Comm", "FitResult", "JFError", "curve_fit", "curve_fit_batch", "graph_cache_clear", "jpass", "nparams", "pass_device",
           "residual_pass", "select_step", "trust_region_step"]
