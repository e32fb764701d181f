"""Drop-in name for `hhengine.cortex`: the recurrent cortex of BASELINE config 5
lives in `network.py` (device network, persistent kernel, sharding); this
module re-exports the reference module's public names (cortex.py:28-464) so
`from hhengine.cortex import run_network` becomes
`from paper_2601_21407_b200.cortex import run_network`."""

from .network import (  # noqa: F401
    REST_CONFIG,
    THALAMIC_CONFIG,
    BackgroundSpec,
    CortexConfig,
    NetworkState,
    NetworkTopology,
    PopulationSpec,
    SpikeBuffer,
    SpikeRecord,
    background_sample,
    build_network,
    init_network_state,
    make_background,
    rest_state_run,
    run_network,
    step_network,
    thalamic_stimulus_run,
)

__all__ = ["REST_CONFIG", "THALAMIC_CONFIG", "BackgroundSpec", "CortexConfig", "NetworkState", "NetworkTopology",
           "PopulationSpec", "SpikeBuffer", "SpikeRecord", "background_sample", "build_network",
           "init_network_state", "make_background", "rest_state_run", "run_network", "step_network",
           "thalamic_stimulus_run"]
