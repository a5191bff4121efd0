"""Domain randomisation / observation noise (reference randomize.py).

Placeholder until the device implementation lands: configurations that ask
for it fail loudly instead of silently running without it.
"""


def check_supported(cfg):
    raise NotImplementedError("EnvConfig.randomize / obs_noise: device domain randomisation is not "
                              "available in this build yet")
