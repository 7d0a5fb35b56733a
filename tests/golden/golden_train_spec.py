"""Inputs of the train() golden (train_run.npz): shared by make_golden.py and
tests/test_dropin_train_golden.py."""

TRAIN_SPEC = dict(n_points=1500, n_features=200, n_labels=2000, labels_per_point=3, noise_level=0.05, seed=21)
TRAIN_CONFIG = dict(epochs=4, batch_size=64, lr_encoder=0.01, lr_classifier=0.05, warmup_steps=5, dropout=0.0,
                    weight_decay_classifier=1e-4, k_r=24, k_h=8, k_p=3, tau_s=2, tau_r=1, strategy="Mixture",
                    seed=0, eval_every=2, embed_dim=128)
